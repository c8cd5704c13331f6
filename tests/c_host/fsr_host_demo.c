/* A C host driving libfsr through include/fsr.h only -- the binding a
 * non-Python caller of the reference's offline + online functions would use
 * (INTEGRATION.md section 2).  Reads a CSR adjacency (normalised W) and one
 * observation vector from a binary file, runs decompose (spectral.py:297-309),
 * sparsify (:269-294) and filter + rank (ranking.py:229-255, 390-395), and
 * writes the eigenvalues, eta, the kept count and the top-k.
 *
 *   fsr_host_demo in.bin out.bin r p q tau topk
 *
 * in.bin : int64 n, nnz, ny; int64 indptr[n+1]; int32 indices[nnz];
 *          float64 data[nnz]; int64 y_idx[ny]; float64 y_val[ny];
 *          float64 w[r] (transfer values h(lambda), computed by the caller
 *          after decompose in a real host; here supplied for the check)
 * out.bin: float64 lam[r]; float64 eta_sparse[n]; int64 kept;
 *          int64 top_idx[topk]; float64 top_val[topk]
 * Test infrastructure (tests/test_gpu_c_host.py). */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "fsr.h"

#define CK(x)                                                                    \
  do {                                                                           \
    int _s = (x);                                                                \
    if (_s) {                                                                    \
      fprintf(stderr, "%s failed: %d (%s)\n", #x, _s, ctx ? fsr_last_error(ctx) : ""); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

static void* up(const void* h, size_t bytes) {
  void* d = NULL;
  if (cudaMalloc(&d, bytes ? bytes : 1) != cudaSuccess) return NULL;
  if (bytes) cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
  return d;
}

int main(int argc, char** argv) {
  fsr_ctx* ctx = NULL;
  if (argc != 8) {
    fprintf(stderr, "usage: %s in.bin out.bin r p q tau topk\n", argv[0]);
    return 2;
  }
  const int64_t r = atoll(argv[3]), p = atoll(argv[4]), tau = atoll(argv[6]), topk = atoll(argv[7]);
  const int q = atoi(argv[5]);
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 2;
  int64_t hdr[3];
  if (fread(hdr, 8, 3, f) != 3) return 2;
  const int64_t n = hdr[0], nnz = hdr[1], ny = hdr[2];
  int64_t* indptr = malloc(8 * (n + 1));
  int32_t* indices = malloc(4 * nnz);
  double* data = malloc(8 * nnz);
  int64_t* y_idx = malloc(8 * ny);
  double* y_val = malloc(8 * ny);
  double* w = malloc(8 * r);
  if (fread(indptr, 8, n + 1, f) != (size_t)(n + 1) || fread(indices, 4, nnz, f) != (size_t)nnz ||
      fread(data, 8, nnz, f) != (size_t)nnz || fread(y_idx, 8, ny, f) != (size_t)ny ||
      fread(y_val, 8, ny, f) != (size_t)ny || fread(w, 8, r, f) != (size_t)r)
    return 2;
  fclose(f);

  CK(fsr_ctx_create(0, &ctx));
  int64_t* d_indptr = up(indptr, 8 * (n + 1));
  int32_t* d_indices = up(indices, 4 * nnz);
  double* d_data = up(data, 8 * nnz);
  double *U, *eta, *eta_s;
  cudaMalloc((void**)&U, 8 * n * r);
  cudaMalloc((void**)&eta, 8 * n);
  cudaMalloc((void**)&eta_s, 8 * n);
  double* lam = malloc(8 * r);

  /* decompose(A, r, p, q, seed=0) in the fp64 parity mode (flags 0: the reference's schedule) */
  CK(fsr_decompose(ctx, FSR_F64, n, d_indptr, d_indices, d_data, r, p, q, 0, 0, lam, U, r, eta));
  /* sparsify(dec, tau) */
  uint64_t T;
  int64_t ties, keep;
  CK(fsr_sparsify_select(ctx, FSR_F64, n, r, U, r, tau, &T, &ties, &keep));
  int64_t* u_indptr;
  int32_t* u_indices;
  double* u_values;
  cudaMalloc((void**)&u_indptr, 8 * (n + 1));
  cudaMalloc((void**)&u_indices, 4 * (keep ? keep : 1));
  cudaMalloc((void**)&u_values, 8 * (keep ? keep : 1));
  int64_t kept = 0;
  CK(fsr_sparsify_apply(ctx, FSR_F64, n, r, U, r, T, ties, u_indptr, u_indices, u_values, eta_s, &kept));
  /* filter + rank for one observation vector */
  int64_t yp[2] = {0, ny};
  int64_t* d_yp = up(yp, 16);
  int64_t* d_yi = up(y_idx, 8 * ny);
  double* d_yv = up(y_val, 8 * ny);
  double* d_w = up(w, 8 * r);
  void* ws;
  cudaMalloc(&ws, fsr_filter_workspace_bytes(FSR_F64, n, r, 1, 0));
  int64_t* d_ti;
  double* d_tv;
  cudaMalloc((void**)&d_ti, 8 * topk);
  cudaMalloc((void**)&d_tv, 8 * topk);
  CK(fsr_filter_batch(ctx, FSR_F64, n, r, 1, u_indptr, u_indices, u_values, NULL, 0, d_w, eta_s, 1, d_yp, d_yi, d_yv,
                      1, ws, NULL, topk, d_ti, d_tv));
  CK(fsr_synchronize(ctx));
  int64_t* ti = malloc(8 * topk);
  double* tv = malloc(8 * topk);
  double* h_eta = malloc(8 * n);
  cudaMemcpy(ti, d_ti, 8 * topk, cudaMemcpyDeviceToHost);
  cudaMemcpy(tv, d_tv, 8 * topk, cudaMemcpyDeviceToHost);
  cudaMemcpy(h_eta, eta_s, 8 * n, cudaMemcpyDeviceToHost);
  f = fopen(argv[2], "wb");
  fwrite(lam, 8, r, f);
  fwrite(h_eta, 8, n, f);
  fwrite(&kept, 8, 1, f);
  fwrite(ti, 8, topk, f);
  fwrite(tv, 8, topk, f);
  fclose(f);
  printf("schedule: %s\nkept %lld\n", fsr_schedule_trace(ctx), (long long)kept);
  fsr_ctx_destroy(ctx);
  return 0;
}
