/*
 * Plain-C use of the C ABI (include/mpid.h) — no Python, no PyTorch: a rank-k
 * mixed-precision ID (Algorithm 2) of a synthetic m x n matrix whose
 * columns j >= r are exact combinations of the first r (so the rank-r ID is exact; a
 * larger k would make A_D(:, I) rank deficient: ID_ERR_DEGENERATE).
 *
 *   gcc -O2 examples/id_c_example.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2012_00706_b200 -lmpid -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2012_00706_b200 -o id_c_example && ./id_c_example
 *
 * Prints k_out, the first pivots, the relative Frobenius error, and exits 0 when the
 * error is below 1e-6.
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "mpid.h"

#define CHECK(call)                                                              \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess) {                                                     \
      fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));                \
      return 2;                                                                  \
    }                                                                            \
  } while (0)

static unsigned long long rng = 88172645463325252ull;
static double urand(void) {   /* xorshift64: a reproducible input, not part of the method */
  rng ^= rng << 13;
  rng ^= rng >> 7;
  rng ^= rng << 17;
  return (double)(rng >> 11) * (1.0 / 9007199254740992.0) - 0.5;
}

int main(void) {
  const int64_t m = 8192, n = 256;
  const int r = 24, k = 24;
  double* A = (double*)malloc(sizeof(double) * m * n);
  double* C = (double*)malloc(sizeof(double) * r * n);
  if (!A || !C) return 2;
  for (int64_t i = 0; i < m * r; ++i) A[i] = urand();               /* columns 0..r-1 */
  for (int64_t i = 0; i < (int64_t)r * n; ++i) C[i] = urand();
  for (int64_t j = r; j < n; ++j)                                    /* A(:, j) = A(:, :r) C(:, j) */
    for (int64_t i = 0; i < m; ++i) {
      double s = 0.0;
      for (int l = 0; l < r; ++l) s += A[l * m + i] * C[j * r + l];
      A[j * m + i] = s;
    }

  double *dA = NULL, *dP = NULL;
  void* ws = NULL;
  CHECK(cudaMalloc((void**)&dA, sizeof(double) * m * n));
  CHECK(cudaMemcpy(dA, A, sizeof(double) * m * n, cudaMemcpyHostToDevice));
  const size_t wsb = id_workspace_bytes(m, n, k, 0, ID_FP32, 0);
  CHECK(cudaMalloc(&ws, wsb));
  CHECK(cudaMalloc((void**)&dP, sizeof(double) * k * n));

  id_handle h = NULL;
  id_status s = id_create(&h, dA, m, m, 0, n, m, ws, wsb, NULL, 0, 1, NULL);
  if (s != ID_OK) { fprintf(stderr, "id_create: %d\n", (int)s); return 1; }
  int32_t kout = 0;
  int32_t piv[64];
  s = id_qrcp_lowprec(h, ID_FP16, ID_SCALE_POW2, k, 0.0, NULL, &kout, piv);
  if (s != ID_OK && s != ID_ERR_UNDERFLOW) { fprintf(stderr, "qrcp: %s\n", id_last_error(h)); return 1; }
  s = id_coeffs_fp64(h, ID_COEF_LSQ, dP, kout);
  if (s != ID_OK) { fprintf(stderr, "coeffs: %s\n", id_last_error(h)); return 1; }
  double abs_e = 0.0, rel_e = 0.0;
  s = id_error(h, &abs_e, &rel_e);
  if (s != ID_OK) { fprintf(stderr, "error: %s\n", id_last_error(h)); return 1; }
  printf("%s\nk_out = %d, first pivots:", id_version(), kout);
  for (int i = 0; i < 8 && i < kout; ++i) printf(" %d", piv[i]);
  printf("\nrelative Frobenius error = %.3e\n", rel_e);
  id_destroy(h);
  cudaFree(dA);
  cudaFree(dP);
  cudaFree(ws);
  free(A);
  free(C);
  return rel_e < 1e-6 ? 0 : 1;
}
