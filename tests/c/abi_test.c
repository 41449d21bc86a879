/*
 * abi_test.c -- a plain C program against include/bspmm.h (no Python, no
 * torch): the C ABI as a C user sees it (§2e "a small C++
 * ABI test").  Links libbspmm.so, and liboracle.so as the independent
 * reference (test infrastructure; the library never sees it).
 *
 *   abi_test cpu   host-only entry points and argument checking (no GPU)
 *   abi_test gpu   + one small batch through bspmm_build_offsets, bspmm_csr,
 *                  bspmm_coo and bspmm_csr_host on device 0, bitwise against
 *                  the oracle's fp32 storage-order sum (O3')
 *
 * Exit status 0 and a final "ok" line on success.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "bspmm.h"

/* oracle/oracle.c (O1, O3', O4) */
int oracle_offsets(int64_t batch, const int32_t* sizes, int64_t* out);
int oracle_spmm_f32(int64_t batch, int32_t k, const int64_t* row_off, const int32_t* sizes, const int32_t* row_ptr,
                    const int32_t* col, const float* vals, const float* B, int64_t ldb, float* C, int64_t ldc);
int oracle_partition(int64_t batch, const int64_t* nnz_off, int32_t k, int32_t parts, int32_t* split);

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static uint32_t next_u32(void) { /* splitmix64 */
  uint64_t z = (rng_state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return (uint32_t)((z ^ (z >> 31)) >> 32);
}
/* U[-1, 1) on the 2^-23 grid */
static float next_val(void) { return (float)((int32_t)(next_u32() >> 8) - (1 << 23)) / (float)(1 << 23); }

static void cpu_checks(void) {
  /* status strings */
  CHECK(strcmp(bspmm_status_string(BSPMM_SUCCESS), "BSPMM_SUCCESS") == 0);
  CHECK(strcmp(bspmm_status_string(BSPMM_ERROR_INDEX), "BSPMM_ERROR_INDEX") == 0);
  CHECK(strcmp(bspmm_status_string((bspmm_status_t)99), "BSPMM_UNKNOWN_STATUS") == 0);
  /* the paper's subWarp rule */
  const int32_t nb[] = {0, 1, 2, 3, 5, 16, 17, 64, 512};
  const int32_t sw[] = {0, 1, 2, 4, 8, 16, 32, 32, 32};
  for (int i = 0; i < 9; ++i) CHECK(bspmm_subwarp(nb[i]) == sw[i]);
  /* partition: hand example (T = 40 over 2 parts: P_2 * 2 = 40 >= 40) and the oracle */
  const int64_t nnz_off[] = {0, 10, 20, 30, 40};
  int32_t split[3] = {-1, -1, -1}, ref[3];
  CHECK(bspmm_partition(4, nnz_off, 1, 2, split) == BSPMM_SUCCESS);
  CHECK(split[0] == 0 && split[1] == 2 && split[2] == 4);
  for (int parts = 1; parts <= 8; ++parts) {
    int64_t off[65];
    off[0] = 0;
    for (int i = 0; i < 64; ++i) off[i + 1] = off[i] + (next_u32() % 50);
    int32_t a[9], b[9];
    CHECK(bspmm_partition(64, off, 256, parts, a) == BSPMM_SUCCESS);
    CHECK(oracle_partition(64, off, 256, parts, b) == 0);
    CHECK(memcmp(a, b, sizeof(int32_t) * (parts + 1)) == 0);
  }
  CHECK(bspmm_partition(4, nnz_off, 1, 0, ref) == BSPMM_ERROR_INVALID_VALUE);
  /* plan: config 5's shape on a 148-SM B200 */
  bspmm_plan_t p;
  CHECK(bspmm_plan(256, 65536, 1, 60, 200, 148, 232448, 0, 0, 0, 0, &p) == BSPMM_SUCCESS);
  CHECK(p.kt > 0 && 256 % p.kt == 0 && p.tiles * p.kt == 256 && p.vec == 1);
  CHECK(p.grid >= 1 && p.grid <= 148 * 4 && p.units == 65536LL * p.tiles);
  CHECK(p.smem_bytes <= 232448);
  CHECK(bspmm_plan(0, 1, 1, 0, 0, 148, 232448, 0, 0, 0, 0, &p) != BSPMM_SUCCESS);
  /* argument checking needs no device */
  CHECK(bspmm_create(NULL, 0, NULL, 0) == BSPMM_ERROR_INVALID_VALUE);
  CHECK(bspmm_destroy(NULL) == BSPMM_SUCCESS);
  CHECK(bspmm_csr(NULL, 1, 4, NULL, NULL, NULL, NULL, NULL, NULL, 4, NULL, 4) == BSPMM_ERROR_INVALID_VALUE);
  CHECK(bspmm_sync(NULL) == BSPMM_ERROR_INVALID_VALUE);
  CHECK(bspmm_launch_count(NULL) == -1);
}

/* a small batch: 5 graphs of 0..40 nodes, 0..4 entries per row (duplicates
 * allowed, arbitrary order), k = 24 */
enum { BATCH = 5, K = 24 };

static void gpu_checks(void) {
  int32_t sizes[BATCH] = {7, 0, 40, 1, 33};
  int64_t row_off[BATCH + 1];
  CHECK(oracle_offsets(BATCH, sizes, row_off) == 0);
  const int64_t N = row_off[BATCH];
  int32_t* row_ptr = malloc(sizeof(int32_t) * (N + 1));
  int32_t* col = malloc(sizeof(int32_t) * N * 4);
  float* vals = malloc(sizeof(float) * N * 4);
  int32_t* coo = malloc(sizeof(int32_t) * N * 8);
  float* B = malloc(sizeof(float) * N * K);
  float* C = malloc(sizeof(float) * N * K);
  float* Cref = malloc(sizeof(float) * N * K);
  int64_t nnz_off[BATCH + 1];
  int32_t e = 0;
  row_ptr[0] = 0;
  nnz_off[0] = 0;
  for (int i = 0; i < BATCH; ++i) {
    for (int r = 0; r < sizes[i]; ++r) {
      const int d = (int)(next_u32() % 5);
      for (int q = 0; q < d; ++q, ++e) {
        col[e] = (int32_t)(next_u32() % (uint32_t)sizes[i]);
        vals[e] = next_val();
        coo[2 * e] = r;
        coo[2 * e + 1] = col[e];
      }
      row_ptr[row_off[i] + r + 1] = e;
    }
    nnz_off[i + 1] = e;
  }
  const int32_t NNZ = e;
  for (int64_t q = 0; q < N * K; ++q) B[q] = next_val();
  CHECK(oracle_spmm_f32(BATCH, K, row_off, NULL, row_ptr, col, vals, B, K, Cref, K) == 0);

  bspmm_handle_t h = NULL;
  CHECK(bspmm_create(&h, 0, NULL, 0) == BSPMM_SUCCESS);
  if (!h) return;
  int32_t *d_sizes, *d_rp, *d_col, *d_coo;
  int64_t *d_ro, *d_no;
  float *d_vals, *d_B, *d_C;
  CHECK(cudaMalloc((void**)&d_sizes, sizeof sizes) == cudaSuccess);
  CHECK(cudaMalloc((void**)&d_ro, sizeof row_off) == cudaSuccess);
  CHECK(cudaMalloc((void**)&d_no, sizeof nnz_off) == cudaSuccess);
  CHECK(cudaMalloc((void**)&d_rp, sizeof(int32_t) * (N + 1)) == cudaSuccess);
  CHECK(cudaMalloc((void**)&d_col, sizeof(int32_t) * (NNZ + 1)) == cudaSuccess);
  CHECK(cudaMalloc((void**)&d_coo, sizeof(int32_t) * 2 * (NNZ + 1)) == cudaSuccess);
  CHECK(cudaMalloc((void**)&d_vals, sizeof(float) * (NNZ + 1)) == cudaSuccess);
  CHECK(cudaMalloc((void**)&d_B, sizeof(float) * N * K) == cudaSuccess);
  CHECK(cudaMalloc((void**)&d_C, sizeof(float) * N * K) == cudaSuccess);
  cudaMemcpy(d_sizes, sizes, sizeof sizes, cudaMemcpyHostToDevice);
  cudaMemcpy(d_no, nnz_off, sizeof nnz_off, cudaMemcpyHostToDevice);
  cudaMemcpy(d_rp, row_ptr, sizeof(int32_t) * (N + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(d_col, col, sizeof(int32_t) * NNZ, cudaMemcpyHostToDevice);
  cudaMemcpy(d_coo, coo, sizeof(int32_t) * 2 * NNZ, cudaMemcpyHostToDevice);
  cudaMemcpy(d_vals, vals, sizeof(float) * NNZ, cudaMemcpyHostToDevice);
  cudaMemcpy(d_B, B, sizeof(float) * N * K, cudaMemcpyHostToDevice);

  /* a-1: offsets on the device, bit-exact */
  int64_t ro_dev[BATCH + 1];
  CHECK(bspmm_build_offsets(h, BATCH, d_sizes, d_ro) == BSPMM_SUCCESS);
  CHECK(bspmm_sync(h) == BSPMM_SUCCESS);
  cudaMemcpy(ro_dev, d_ro, sizeof ro_dev, cudaMemcpyDeviceToHost);
  CHECK(memcmp(ro_dev, row_off, sizeof row_off) == 0);
  /* CSR, with row offsets and with sizes only */
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(d_C, 0xff, sizeof(float) * N * K);
    CHECK(bspmm_csr(h, BATCH, K, mode ? NULL : d_ro, mode ? d_sizes : NULL, d_rp, d_col, d_vals, d_B, K, d_C, K) ==
          BSPMM_SUCCESS);
    CHECK(bspmm_sync(h) == BSPMM_SUCCESS);
    cudaMemcpy(C, d_C, sizeof(float) * N * K, cudaMemcpyDeviceToHost);
    CHECK(memcmp(C, Cref, sizeof(float) * N * K) == 0);
  }
  /* COO / SparseTensor (each row's entries were generated in a random column
   * order; the canonical CSR keeps duplicates in input order) */
  cudaMemset(d_C, 0xff, sizeof(float) * N * K);
  CHECK(bspmm_coo(h, BATCH, K, d_ro, NULL, d_no, d_coo, d_vals, d_B, K, d_C, K, N, NNZ, NULL, NULL, NULL) ==
        BSPMM_SUCCESS);
  CHECK(bspmm_sync(h) == BSPMM_SUCCESS);
  cudaMemcpy(C, d_C, sizeof(float) * N * K, cudaMemcpyDeviceToHost);
  for (int64_t q = 0; q < N * K; ++q) /* within the per-element bound: sum order may differ per row */
    CHECK(C[q] == C[q] && (C[q] - Cref[q] <= 1e-5f && Cref[q] - C[q] <= 1e-5f));
  /* end to end on host buffers */
  memset(C, 0xff, sizeof(float) * N * K);
  CHECK(bspmm_csr_host(h, BATCH, K, sizes, row_ptr, col, vals, B, C, N, NNZ) == BSPMM_SUCCESS);
  CHECK(memcmp(C, Cref, sizeof(float) * N * K) == 0);
  /* argument errors are reported, not thrown, and leave the handle usable */
  CHECK(bspmm_csr(h, -1, K, d_ro, NULL, d_rp, d_col, d_vals, d_B, K, d_C, K) == BSPMM_ERROR_INVALID_VALUE);
  CHECK(strlen(bspmm_last_error_string(h)) > 0);
  CHECK(bspmm_csr(h, BATCH, K, d_ro, NULL, d_rp, d_col, d_vals, d_B, K, (float*)d_B, K) ==
        BSPMM_ERROR_INVALID_VALUE);
  CHECK(bspmm_launch_count(h) > 0);
  CHECK(bspmm_destroy(h) == BSPMM_SUCCESS);
  cudaFree(d_sizes), cudaFree(d_ro), cudaFree(d_no), cudaFree(d_rp), cudaFree(d_col), cudaFree(d_coo);
  cudaFree(d_vals), cudaFree(d_B), cudaFree(d_C);
  free(row_ptr), free(col), free(vals), free(coo), free(B), free(C), free(Cref);
}

int main(int argc, char** argv) {
  const int gpu = argc > 1 && strcmp(argv[1], "gpu") == 0;
  cpu_checks();
  if (gpu) {
    gpu_checks();
  } else {
    bspmm_handle_t h = NULL;
    const bspmm_status_t s = bspmm_create(&h, 0, NULL, 0);
    CHECK(s == BSPMM_ERROR_NOT_SUPPORTED || s == BSPMM_SUCCESS); /* no device here, or a B200 */
    bspmm_destroy(h);
  }
  if (failures) {
    fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  printf("ok\n");
  return 0;
}
