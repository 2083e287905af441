/*
 * nrmf.h -- C ABI of the B200-native xNRMF library (libnrmf.so).
 *
 * xNRMF (arXiv 2509.06220, "Recursive vectorized computation of the Frobenius
 * norm", cited as P:<line of /root/reference/PAPER.md>) computes ||x||_F of a
 * real fp32/fp64 array without squaring any element: partial norms of two
 * disjoint parts are combined by a hypotenuse function, e:hr,
 * recursively down a fixed binary tree (Listing 1), with the
 * branch-free v1_hypot of Listing 2 at every node:
 *
 *     X=|x|, Y=|y|, m=fmin(X,Y), M=fmax(X,Y), q=m/M, Q=fmax(q,0),
 *     S=fma(Q,Q,1), s=sqrt(S), h=M*s          (each step IEEE round-to-nearest)
 *
 * The tree is the frozen "tile-lane tree" (tree version 1):
 * fp64 uses p=64 lanes x J=64, fp32 p=128 lanes x J=32, tile T=4096 elements.
 * Element i of tile tau=i/T sits in lane l=(i%T)%p at depth position
 * j=(i%T)/p; each lane reduces its strided subsequence as in Z;
 * lanes, tiles and ranks are then combined by balanced trees in contiguous
 * order (the A-shaped final reduction of P:962-967, with v1_hypot).  The tail
 * is zero-padded (the paper's masked tail) to a power-of-two number
 * of tiles.  Results therefore do not depend on the launch geometry, the
 * alignment of x, the number of GPUs, or the run: they are bitwise
 * reproducible and bit-exact with the same-tree CPU oracle.
 *
 * Conventions for every call below
 *  - Pointers named x, A, out, col_norms, frob, ws are DEVICE pointers (or
 *    managed memory) unless the name says host_; they must be naturally aligned
 *    (4 B for float, 8 B for double), otherwise NRMF_EALIGN.  16-byte aligned
 *    inputs use 128-bit loads; other inputs give identical bits, more slowly.
 *  - stream is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call is asynchronous and ordered on stream; the library never
 *    synchronizes the device, never allocates device memory and never prints.
 *  - ws is a caller-owned device workspace of at least the size returned by the
 *    matching *_workspace_bytes call, 16-byte aligned (cudaMalloc and torch
 *    allocations are; NRMF_EALIGN otherwise).  Its contents on entry do not matter
 *    (the call clears the few bytes of arrival counters it uses, on stream,
 *    before its kernel).  A workspace must not be shared by calls that may
 *    run concurrently (distinct workspaces and streams make the calls
 *    reentrant and thread-safe).
 *  - Status is returned at enqueue time: NRMF_EINVAL for n<0 / null pointers /
 *    bad shapes, NRMF_EALIGN, NRMF_EWORKSPACE, NRMF_ESHARD, NRMF_ECUDA for a
 *    launch error (cudaGetLastError), NRMF_ENCCL for an NCCL error.
 *    Asynchronous device faults surface at the caller's next synchronization.
 *  - Semantics: n=0 gives +0; results are in the input precision; non-finite
 *    inputs follow Listing 2 literally (fmin/fmax ignore a NaN operand, so
 *    v1_hypot(NaN,0)=+0 and NaN is returned only when both operands are NaN;
 *    any +-inf that reaches a node gives +inf).  Finite inputs never overflow
 *    or underflow spuriously (only if the true norm exceeds the format).
 */
#ifndef NRMF_H
#define NRMF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    NRMF_OK = 0,
    NRMF_EINVAL = 1,      /* invalid argument (negative size, null pointer, bad shape) */
    NRMF_EALIGN = 2,      /* pointer not aligned to its element size                   */
    NRMF_EWORKSPACE = 3,  /* ws_bytes smaller than required                            */
    NRMF_ESHARD = 4,      /* (offset,count) is not the canonical shard of this rank    */
    NRMF_ECUDA = 5,       /* CUDA launch / runtime error                               */
    NRMF_ENCCL = 6        /* NCCL error, or NCCL could not be loaded                   */
} nrmf_status;

/* Flags of the *_ex_* calls.
 * NRMF_TOP_CR: every node ABOVE the tile level (warp groups, grid steps,
 *   column trees, the Frobenius tree over columns, host chunks, ranks) uses
 *   the correctly rounded hypot cr_hypot(a,b) = RN(sqrt(a^2+b^2)) instead of
 *   v1_hypot -- the paper's recommended final reduction "Z with A"
 *   (A_x = R with cr_hypot).  The tiles keep v1_hypot.
 *   Relative error bound: ((1+eps'+)^lg T * (1+eps)^lg(P2) - 1)/eps, e.g.
 *   36 + 18 = 54 eps at n = 2^30 fp64 (< 64: the 64-eps target becomes a
 *   theorem).  cr_hypot follows IEEE 754 hypot for specials
 *   (+inf if either operand is infinite, else NaN if either is NaN). */
#define NRMF_TOP_CR 1

/* NRMF_WS_CLEAN: the caller guarantees that the workspace's arrival counters
 *   are zero on entry: ws was zero-filled before its first call and has since
 *   been used only by calls with identical arguments (e.g. the warm-up and the
 *   replays of one captured CUDA graph), each completed before the next began.
 *   Every completed call leaves its counters zero, so the guarantee carries
 *   over; the call then skips its counter memset and is a single kernel (one
 *   graph node).  Without it (the default) the contents of ws never matter.
 *   Ignored by the host-input calls, which always clear their counters. */
#define NRMF_WS_CLEAN 2

/* Human-readable name of a status code (static string). */
const char *nrmf_status_str(int status);

/* Version of the frozen reduction tree; bumps whenever (p, J, T) change. */
int nrmf_tree_version(void);

/* Tree constants for elem_bytes 8 (fp64) or 4 (fp32): lanes p, J, tile T. */
int nrmf_tree_params(int elem_bytes, int *lanes, int *J, int *tile);

/* ------------------------------------------------------------------------ */
/* One vector: out[0] = ||x[0..n)||_F   (xNRMF; e:F P:55-62)      */
/* ------------------------------------------------------------------------ */
size_t nrmf_workspace_bytes(int64_t n, int elem_bytes);
int nrmf_d(int64_t n, const double *x, double *out, void *ws, size_t ws_bytes, void *stream);
int nrmf_s(int64_t n, const float *x, float *out, void *ws, size_t ws_bytes, void *stream);

/* The same with flags (NRMF_TOP_CR | NRMF_WS_CLEAN or 0); flags 0 is bitwise
 * nrmf_[ds] (NRMF_WS_CLEAN never changes a result, only the launches). */
int nrmf_ex_d(int64_t n, const double *x, double *out, int flags, void *ws, size_t ws_bytes, void *stream);
int nrmf_ex_s(int64_t n, const float *x, float *out, int flags, void *ws, size_t ws_bytes, void *stream);

/* Complex view (e:F: the real and imaginary parts are just more
 * elements): ||z||_F of count interleaved (re,im) pairs; bitwise identical to
 * nrmf_[ds](2*count, (real*)z, ...). */
int nrmf_z_d(int64_t count, const double *z, double *out, void *ws, size_t ws_bytes, void *stream);
int nrmf_z_s(int64_t count, const float *z, float *out, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------ */
/* Column norms of a column-major rows x cols matrix A (leading dimension     */
/* ld >= rows, element (i,j) at A[i + j*ld]) -- the inner sum of e:F         */
/* (P:55-59).  col_norms[j] is bitwise nrmf of column j (length rows); frob  */
/* (nullable) is the balanced tree over the cols column norms padded with +0 */
/* to a power of two.  rows=0 gives zero column norms; cols=0 gives frob=+0. */
/* ------------------------------------------------------------------------ */
size_t nrmf_cols_workspace_bytes(int64_t rows, int64_t cols, int elem_bytes);
int nrmf_cols_d(int64_t rows, int64_t cols, int64_t ld, const double *A, double *col_norms,
                double *frob, void *ws, size_t ws_bytes, void *stream);
int nrmf_cols_s(int64_t rows, int64_t cols, int64_t ld, const float *A, float *col_norms,
                float *frob, void *ws, size_t ws_bytes, void *stream);
int nrmf_cols_ex_d(int64_t rows, int64_t cols, int64_t ld, const double *A, double *col_norms,
                   double *frob, int flags, void *ws, size_t ws_bytes, void *stream);
int nrmf_cols_ex_s(int64_t rows, int64_t cols, int64_t ld, const float *A, float *col_norms,
                   float *frob, int flags, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------ */
/* Host-resident input (pinned memory for overlap): streams host_x through a  */
/* device staging ring inside ws, overlapping the H2D copies with the        */
/* per-chunk reductions; chunks are aligned subtrees of the same tree, so     */
/* *host_out is bitwise equal to nrmf_[ds] of the same data.  host_out is    */
/* written by an async D2H copy on stream: synchronize stream before reading. */
/* ------------------------------------------------------------------------ */
size_t nrmf_host_workspace_bytes(int64_t n, int elem_bytes);
int nrmf_host_d(int64_t n, const double *host_x, double *host_out, void *ws, size_t ws_bytes,
                void *stream);
int nrmf_host_s(int64_t n, const float *host_x, float *host_out, void *ws, size_t ws_bytes,
                void *stream);
int nrmf_host_ex_d(int64_t n, const double *host_x, double *host_out, int flags, void *ws,
                   size_t ws_bytes, void *stream);
int nrmf_host_ex_s(int64_t n, const float *host_x, float *host_out, int flags, void *ws,
                   size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------ */
/* One array sharded contiguously over the `world` ranks of an NCCL          */
/* communicator (e:hr P:216-231: partial norms of disjoint parts combine by  */
/* hypot; contiguous chunks per worker, in a FIXED order).       */
/* Canonical shard: NT = ceil(n_global/T) tiles, P2 = pow2 >= NT; if         */
/* world <= P2 rank r owns tiles [r*P2/world, (r+1)*P2/world), else rank      */
/* r < P2 owns tile r; clipped to n_global.  Each rank reduces its aligned   */
/* subtree, one ncclAllGather of one scalar per rank follows, and every rank */
/* evaluates the top of the same balanced tree: out (device, 1 element) is   */
/* bitwise identical on every rank and equal to nrmf_[ds] of the whole array */
/* on one GPU.  Collective: every rank must call with the same n_global.     */
/* world must be a power of two (NRMF_ESHARD otherwise).                     */
/* ------------------------------------------------------------------------ */
int nrmf_dist_shard(int64_t n_global, int world, int rank, int64_t *offset, int64_t *count);
size_t nrmf_dist_workspace_bytes(int64_t n_global, int world, int elem_bytes);
int nrmf_dist_d(int64_t n_global, int64_t offset, int64_t count, const double *x_local,
                double *out, void *ws, size_t ws_bytes, void *nccl_comm, void *stream);
int nrmf_dist_s(int64_t n_global, int64_t offset, int64_t count, const float *x_local,
                float *out, void *ws, size_t ws_bytes, void *nccl_comm, void *stream);
int nrmf_dist_ex_d(int64_t n_global, int64_t offset, int64_t count, const double *x_local,
                   double *out, int flags, void *ws, size_t ws_bytes, void *nccl_comm, void *stream);
int nrmf_dist_ex_s(int64_t n_global, int64_t offset, int64_t count, const float *x_local,
                   float *out, int flags, void *ws, size_t ws_bytes, void *nccl_comm, void *stream);

/* The two halves of nrmf_dist_[ds], for callers that move the rank values  */
/* themselves (their own collective, MPI, ...) -- and the kernels the NCCL    */
/* and peer-memory paths run:                                                 */
/*  nrmf_dist_local_[ds]: *local_out (device, 1 element) = the value of this  */
/*    rank's aligned subtree (the same tree kernel as nrmf_[ds]; +0 for a     */
/*    rank that owns no data); arguments and workspace as nrmf_dist_[ds],     */
/*    with world/rank given explicitly.                                       */
/*  nrmf_rank_combine_[ds]: *out = the rank tree (the top lg min(world, P2)   */
/*    levels of the global tree) over values[0 .. min(world, P2)) (device, in  */
/*    rank order; P2 = pow2 >= ceil(n_global/T)).  One CTA, no workspace.      */
/* Gathering every rank's local_out in rank order and combining them gives    */
/* bitwise nrmf_[ds] of the whole array (tested through these two calls for   */
/* 2, 4 and 8 ranks on one GPU).                                             */
int nrmf_dist_local_d(int64_t n_global, int world, int rank, int64_t offset, int64_t count,
                      const double *x_local, double *local_out, int flags, void *ws, size_t ws_bytes,
                      void *stream);
int nrmf_dist_local_s(int64_t n_global, int world, int rank, int64_t offset, int64_t count,
                      const float *x_local, float *local_out, int flags, void *ws, size_t ws_bytes,
                      void *stream);
int nrmf_rank_combine_d(int64_t n_global, int world, const double *values, double *out, int flags, void *stream);
int nrmf_rank_combine_s(int64_t n_global, int world, const float *values, float *out, int flags, void *stream);

/* ------------------------------------------------------------------------ */
/* Column norms of a column-major rows x cols_global matrix whose columns are */
/* sharded in blocks over the ranks.  Canonical block: P2c = pow2 */
/* >= cols_global column leaves of the Frobenius tree; if world <= P2c rank r */
/* owns columns [r*P2c/world, (r+1)*P2c/world), else rank r < P2c owns column */
/* r; clipped to cols_global (nrmf_cols_dist_shard).  A_local holds the       */
/* rank's col_count columns (leading dimension ld >= rows), col_norms_local    */
/* receives their norms (bitwise those of nrmf_cols_[ds] on the whole matrix: */
/* a column never spans ranks).  frob (device, 1 element, nullable on every   */
/* rank or on none): the rank's block is an aligned subtree of the Frobenius  */
/* tree (size P2c/world), one ncclAllGather of one scalar per rank follows,   */
/* and every rank evaluates the top levels, so *frob is bitwise identical on  */
/* every rank and equal to nrmf_cols_[ds]'s frob on one GPU.  Collective when */
/* frob is non-null.  flags: NRMF_TOP_CR | NRMF_WS_CLEAN or 0.  world a      */
/* power of two.                                                             */
/* ------------------------------------------------------------------------ */
int nrmf_cols_dist_shard(int64_t cols_global, int world, int rank, int64_t *col_offset, int64_t *col_count);
size_t nrmf_cols_dist_workspace_bytes(int64_t rows, int64_t cols_global, int world, int elem_bytes);
int nrmf_cols_dist_d(int64_t rows, int64_t cols_global, int64_t ld, int64_t col_offset, int64_t col_count,
                     const double *A_local, double *col_norms_local, double *frob, int flags, void *ws,
                     size_t ws_bytes, void *nccl_comm, void *stream);
int nrmf_cols_dist_s(int64_t rows, int64_t cols_global, int64_t ld, int64_t col_offset, int64_t col_count,
                     const float *A_local, float *col_norms_local, float *frob, int flags, void *ws,
                     size_t ws_bytes, void *nccl_comm, void *stream);

/* ------------------------------------------------------------------------ */
/* The rank level through peer memory instead of NCCL: the same  */
/* canonical shards and the same rank tree as nrmf_dist_[ds], but the        */
/* exchange is fused into the tree kernel: the warp that evaluates the rank's */
/* subtree root stores it into every peer's buffer (P2P stores to CUDA-IPC-    */
/* mapped memory over NVLink) with a release flag, waits for every rank's      */
/* value in its own buffer, evaluates the rank tree and writes *out -- one     */
/* kernel per call, no ncclAllGather and no rank-tree launch (P:1077-1084:     */
/* contiguous chunks per worker, combined in a fixed order).  The wait runs    */
/* only after this rank's whole subtree is done (ranks are distinct GPUs).     */
/* Setup (once per rank, collective through the caller's own channel):        */
/*   nrmf_p2p_alloc(&buf) -- nrmf_p2p_buffer_bytes() of device memory,       */
/*     zero-filled (the one allocation the library makes; free it with     */
/*     nrmf_p2p_free);                                                      */
/*   nrmf_p2p_ipc_handle(buf, h) -- 64-byte CUDA IPC handle, all-gathered;    */
/*   nrmf_p2p_open(h_r, &ptr_r) for every other rank r (close: _p2p_close);   */
/*   peers: a DEVICE array of world pointers, peers[r] = rank r's buffer as  */
/*     mapped in this process, peers[rank] = buf.                             */
/* Calls: every rank makes the same sequence of calls; the buffer keeps a    */
/* call counter and two parity halves, so nothing is reset between calls and */
/* a call can be captured in a CUDA graph.  err (device u32, nullable) is set */
/* to 1 if a rank's value did not arrive within ~seconds (out is then NaN     */
/* instead of a hang).  world: a power of two <= 32.                          */
/* Every rank's out has the same bits, equal to nrmf_[ds] on one GPU.         */
/* ------------------------------------------------------------------------ */
size_t nrmf_p2p_buffer_bytes(void);
int nrmf_p2p_alloc(void **buf);
int nrmf_p2p_free(void *buf);
int nrmf_p2p_ipc_handle(const void *buf, char *handle64);
int nrmf_p2p_open(const char *handle64, void **peer_buf);
int nrmf_p2p_close(void *peer_buf);
int nrmf_dist_p2p_d(int64_t n_global, int64_t offset, int64_t count, const double *x_local, double *out,
                    int flags, void *ws, size_t ws_bytes, const void *peers, int world, int rank,
                    unsigned *err, void *stream);
int nrmf_dist_p2p_s(int64_t n_global, int64_t offset, int64_t count, const float *x_local, float *out,
                    int flags, void *ws, size_t ws_bytes, const void *peers, int world, int rank,
                    unsigned *err, void *stream);

/* NCCL bootstrap helpers (libnccl.so.2 is loaded at first use; the process's
 * already-loaded NCCL, e.g. torch's, is reused).  id is 128 bytes: create it
 * on one rank, broadcast it (e.g. through torch.distributed), then call
 * comm_init on every rank with the current CUDA device already selected. */
int nrmf_nccl_unique_id(char *id128);
int nrmf_nccl_comm_init(int world, int rank, const char *id128, void **nccl_comm);
int nrmf_nccl_comm_destroy(void *nccl_comm);

#ifdef __cplusplus
}
#endif

#endif /* NRMF_H */
