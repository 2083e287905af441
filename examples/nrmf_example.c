/*
 * examples/nrmf_example.c -- calling libnrmf.so from plain C (no Python, no
 * torch): ||x||_F of n doubles read from a binary file (or x_i = i+1 if no
 * file is given), computed on the current CUDA device with nrmf_d, and printed
 * as a decimal and as its IEEE-754 bit pattern.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/nrmf_example.c -o nrmf_example \
 *       -L paper_2509_06220_b200 -l:libnrmf.so -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2509_06220_b200 -Wl,-rpath,/usr/local/cuda/lib64
 *   ./nrmf_example [n] [file.f64]
 */
#include <cuda_runtime.h>
#include <inttypes.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "nrmf.h"

#define CK(call)                                                                   \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) {                                                   \
            fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));            \
            return 2;                                                              \
        }                                                                          \
    } while (0)

int main(int argc, char **argv)
{
    const int64_t n = argc > 1 ? strtoll(argv[1], NULL, 10) : 1000003;
    double *h = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    if (!h) return 2;
    if (argc > 2) {
        FILE *f = fopen(argv[2], "rb");
        if (!f || fread(h, sizeof(double), (size_t)n, f) != (size_t)n) {
            fprintf(stderr, "cannot read %" PRId64 " doubles from %s\n", n, argv[2]);
            return 2;
        }
        fclose(f);
    } else {
        for (int64_t i = 0; i < n; ++i) h[i] = (double)(i + 1);
    }
    double *x = NULL, *out = NULL;
    void *ws = NULL;
    const size_t ws_bytes = nrmf_workspace_bytes(n, 8);
    CK(cudaMalloc((void **)&x, (size_t)(n > 0 ? n : 1) * sizeof(double)));
    CK(cudaMalloc((void **)&out, sizeof(double)));
    CK(cudaMalloc(&ws, ws_bytes));
    CK(cudaMemcpy(x, h, (size_t)n * sizeof(double), cudaMemcpyHostToDevice));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    const int st = nrmf_d(n, x, out, ws, ws_bytes, (void *)s);   /* asynchronous on s */
    if (st != NRMF_OK) {
        fprintf(stderr, "nrmf_d: %s\n", nrmf_status_str(st));
        return 1;
    }
    double r = 0.0;
    CK(cudaMemcpyAsync(&r, out, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    uint64_t bits;
    memcpy(&bits, &r, sizeof bits);
    printf("n=%" PRId64 " norm=%.17g bits=%016" PRIx64 " tree_version=%d\n", n, r, bits, nrmf_tree_version());
    cudaFree(x); cudaFree(out); cudaFree(ws); cudaStreamDestroy(s); free(h);
    return 0;
}
