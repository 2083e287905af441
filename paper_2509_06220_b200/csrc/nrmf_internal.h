// nrmf_internal.h -- entry points shared by the translation units of libnrmf.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace nrmf {
// Rank exchange fused into the tree kernel (nrmf_p2p.cuh): the warp that
// evaluates the local root publishes it to the peers, waits for theirs and
// writes the rank tree's root instead.
struct RankExchange {
  char* const* peers;  // device array of world buffer pointers
  unsigned* err;       // nullable
  int world, rank, nr;
};
// Balanced tree over p2 tiles of x[0..n) (zero padded) -> *out (device).
template <typename F>
int tree_eval(int64_t n, const F* x, int64_t p2, F* out, void* ws, size_t ws_bytes, cudaStream_t s,
              int top_cr, const RankExchange* rx = nullptr);
// Balanced tree over vals[0..P) (entries >= nvals are +0) -> *out, one CTA.
template <typename F>
int bal_eval(const F* vals, int64_t nvals, int64_t P, F* out, cudaStream_t s, int top_cr);
// Workspace bytes of tree_eval for a p2-tile tree.
size_t tree_workspace(int64_t p2, size_t esz);
// Column norms + Frobenius tree of size p2cols (a power of two >= cols) over
// them; arguments validated like nrmf_cols_ex_[ds].
template <typename F>
int cols_eval(int64_t rows, int64_t cols, int64_t ld, const F* A, F* col_norms, F* frob, int64_t p2cols,
              int flags, void* ws, size_t ws_bytes, cudaStream_t s);
size_t cols_workspace(int64_t rows, int64_t cols, int64_t p2cols, size_t esz);
}  // namespace nrmf
