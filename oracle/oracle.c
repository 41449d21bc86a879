/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU
 * implementation of what the Batched SpMM hot path computes (arXiv 1903.11409).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_1903_11409_b200/) and includes
 * nothing from it.  Built with -O2 -fopenmp -ffp-contract=off, no fast-math.
 * OpenMP is used only across independent matrices, so results do not depend
 * on the thread count.
 *
 * Functions and the passages they follow:
 *   O1 oracle_offsets      exclusive prefix sum of per-matrix sizes (the
 *                          "list of adjacency matrices ... accumulating the
 *                          pointers"; offsets replace the device
 *                          pointer arrays of PAPER.md:343).
 *   O2 oracle_coo2csr      SparseTensor pairs (unsorted :141) ->
 *                          CSR rpt/colids/values in canonical
 *                          (row, col, original position) order (R5).
 *   O3 oracle_spmm         C = A B, per-entry semantics of the
 *                          pseudo-code C[rid][j] += val * B[cid][j]
 *                           over the stored entries,
 *                          accumulated in fp64, rounded once to fp32, with the
 *                          per-element bound 1e-5 * sum |a||b| (north_star).
 *   O3' oracle_spmm_f32    the same sum in fp32 as fmaf in CSR storage order
 *                          (PAPER.md:201-205 loop order; R14).
 *   O3s oracle_spmm_rows   O3 for a list of sampled (matrix, row) pairs.
 *   O4 oracle_partition    contiguous split of graphs over G ranks by nnz*k
 *                          prefix (north_star; R25).
 *   O5 oracle_csr_transpose per-matrix A_i^T (backward), canonical
 *                          (row, col, original position) order.
 *   O6 oracle_sddmm        grad_vals[e] = <grad_C[row_e], B[col_e]> in fp64
 *                          with bound 1e-5 * sum |d||b| (adjoint of C = A B,
 *                          SPEC.md:178-186).
 *   O7 oracle_gcn_layer    Y = sum_ch A_ch (X W_ch + 1 bias_ch^T) (PAPER.md Fig.
 *                          algo:graph_conv_batched, Eq. (2)), fp64, with the
 *                          magnitude sum that scales its tolerance.
 *
 * Pins (tests/test_oracle_pins.py): dense brute force A@B (numpy fp64) on
 * >=1000 tiny batches, identity -> C == B, SPEC.md:140 example, zero rows,
 * linearity in B, integer-valued exactness, COO permutation invariance and
 * brute-force sorted(), partition invariants and closed forms; backward:
 * central finite differences of L = sum(C * G), dense A^T brute force,
 * SPEC.md:177/:185 worked examples.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* n_i: sizes[i] when given, else the packed difference of row_off */
static int64_t rows_of(const int64_t* row_off, const int32_t* sizes, int64_t i) {
  return sizes ? (int64_t)sizes[i] : row_off[i + 1] - row_off[i];
}

/* O1 */
int oracle_offsets(int64_t batch, const int32_t* sizes, int64_t* out) {
  if (batch < 0) return 1;
  out[0] = 0;
  for (int64_t i = 0; i < batch; ++i) out[i + 1] = out[i] + (int64_t)sizes[i];
  return 0;
}

/* O2 */
typedef struct { int32_t row, col; int64_t pos; } trip_t;
static int cmp_trip(const void* a, const void* b) {
  const trip_t* x = (const trip_t*)a;
  const trip_t* y = (const trip_t*)b;
  if (x->row != y->row) return x->row < y->row ? -1 : 1;
  if (x->col != y->col) return x->col < y->col ? -1 : 1;
  return (x->pos > y->pos) - (x->pos < y->pos);
}

int oracle_coo2csr(int64_t batch, const int64_t* row_off, const int32_t* sizes,
                   const int64_t* nnz_off, const int32_t* idx, const float* vals,
                   int32_t* row_ptr, int32_t* col_out, float* val_out) {
  if (batch < 0) return 1;
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(|:bad)
  for (int64_t i = 0; i < batch; ++i) {
    int64_t n = rows_of(row_off, sizes, i);
    int64_t z0 = nnz_off[i], m = nnz_off[i + 1] - z0;
    trip_t* t = (trip_t*)malloc(sizeof(trip_t) * (size_t)(m > 0 ? m : 1));
    for (int64_t e = 0; e < m; ++e) {
      t[e].row = idx[2 * (z0 + e)];
      t[e].col = idx[2 * (z0 + e) + 1];
      t[e].pos = e;
      if (t[e].row < 0 || t[e].row >= n || t[e].col < 0 || t[e].col >= n) bad = 1;
    }
    qsort(t, (size_t)m, sizeof(trip_t), cmp_trip);
    /* row pointer: count entries per row, then running sum */
    int64_t e = 0;
    for (int64_t r = 0; r < n; ++r) {
      row_ptr[row_off[i] + r] = (int32_t)(z0 + e);
      while (e < m && t[e].row == r) ++e;
    }
    /* padding rows between this matrix and the next own no entries */
    for (int64_t g = row_off[i] + n; g < row_off[i + 1]; ++g) row_ptr[g] = (int32_t)(z0 + m);
    for (int64_t q = 0; q < m; ++q) {
      col_out[z0 + q] = t[q].col;
      val_out[z0 + q] = vals[z0 + t[q].pos]; /* bitwise copy */
    }
    free(t);
  }
  if (batch > 0) row_ptr[row_off[batch]] = (int32_t)nnz_off[batch];
  return bad ? 4 : 0;
}

/* O3: fp64 accumulation, one rounding to fp32, bound = 1e-5 * sum |a||b| */
int oracle_spmm(int64_t batch, int32_t k, const int64_t* row_off, const int32_t* sizes,
                const int32_t* row_ptr, const int32_t* col, const float* vals,
                const float* B, int64_t ldb, float* C, int64_t ldc, double* bound,
                double* C64) {
  if (batch < 0 || k < 0) return 1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < batch; ++i) {
    int64_t n = rows_of(row_off, sizes, i);
    for (int64_t r = 0; r < n; ++r) {
      int64_t g = row_off[i] + r;
      for (int32_t c = 0; c < k; ++c) {
        double acc = 0.0, s = 0.0;
        for (int64_t e = row_ptr[g]; e < row_ptr[g + 1]; ++e) {
          double a = (double)vals[e];
          double b = (double)B[(row_off[i] + col[e]) * ldb + c];
          acc += a * b;
          s += fabs(a) * fabs(b);
        }
        C[g * ldc + c] = (float)acc;
        if (bound) bound[g * ldc + c] = 1e-5 * s;
        if (C64) C64[g * ldc + c] = acc;
      }
    }
  }
  return 0;
}

/* O3': fp32, fmaf in CSR storage order, acc starts at +0.0f */
int oracle_spmm_f32(int64_t batch, int32_t k, const int64_t* row_off, const int32_t* sizes,
                    const int32_t* row_ptr, const int32_t* col, const float* vals,
                    const float* B, int64_t ldb, float* C, int64_t ldc) {
  if (batch < 0 || k < 0) return 1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < batch; ++i) {
    int64_t n = rows_of(row_off, sizes, i);
    for (int64_t r = 0; r < n; ++r) {
      int64_t g = row_off[i] + r;
      for (int32_t c = 0; c < k; ++c) {
        float acc = 0.0f;
        for (int64_t e = row_ptr[g]; e < row_ptr[g + 1]; ++e)
          acc = fmaf(vals[e], B[(row_off[i] + col[e]) * ldb + c], acc);
        C[g * ldc + c] = acc;
      }
    }
  }
  return 0;
}

/* O3s: O3 for sampled rows; (mat[s], r[s]) -> out[s*k + c], bound[s*k + c] */
int oracle_spmm_rows(int64_t nsamp, const int64_t* mat, const int32_t* rloc, int32_t k,
                     const int64_t* row_off, const int32_t* row_ptr, const int32_t* col,
                     const float* vals, const float* B, int64_t ldb, float* out, double* bound) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t s = 0; s < nsamp; ++s) {
    int64_t i = mat[s];
    int64_t g = row_off[i] + rloc[s];
    for (int32_t c = 0; c < k; ++c) {
      double acc = 0.0, t = 0.0;
      for (int64_t e = row_ptr[g]; e < row_ptr[g + 1]; ++e) {
        double a = (double)vals[e];
        double b = (double)B[(row_off[i] + col[e]) * ldb + c];
        acc += a * b;
        t += fabs(a) * fabs(b);
      }
      out[s * k + c] = (float)acc;
      bound[s * k + c] = 1e-5 * t;
    }
  }
  return 0;
}

/* O4: cost c_i = nnz_i * k; P_j = sum_{i<j} c_i; T = P_batch.
 * split[0] = 0, split[G] = batch; for 0<r<G: smallest j in [0,batch] with
 * P_j * G >= r * T; if T == 0: split[r] = floor(r * batch / G). */
int oracle_partition(int64_t batch, const int64_t* nnz_off, int32_t k, int32_t parts,
                     int32_t* split) {
  if (batch < 0 || parts < 1 || k < 0) return 1;
  int64_t T = (nnz_off[batch] - nnz_off[0]) * (int64_t)k;
  split[0] = 0;
  split[parts] = (int32_t)batch;
  for (int32_t r = 1; r < parts; ++r) {
    if (T == 0) {
      split[r] = (int32_t)((int64_t)r * batch / parts);
      continue;
    }
    int64_t j = 0;
    while (j < batch && (nnz_off[j] - nnz_off[0]) * (int64_t)k * parts < (int64_t)r * T) ++j;
    split[r] = (int32_t)j;
  }
  return 0;
}

/* ---- backward (NEXT-2): "The Batched SpMM is also applied to
 * backward propagation"; formulas are the standard adjoints of C = A B
 * (SPEC.md:169-186): grad_B = A^T grad_C, grad_vals[e] = <grad_C[row_e], B[col_e]>. */

/* O5 per-matrix transpose of a block-diagonal CSR: entries (r, c, v) of A_i
 * become (c, r, v) of A_i^T, emitted in canonical (row, col, original
 * position) order; absolute row pointers, LOCAL column ids. */
int oracle_csr_transpose(int64_t batch, const int64_t* row_off, const int32_t* sizes,
                         const int32_t* row_ptr, const int32_t* col, const float* vals,
                         int32_t* rowT, int32_t* colT, float* valsT) {
  if (batch < 0) return 1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < batch; ++i) {
    int64_t n = rows_of(row_off, sizes, i);
    int64_t g0 = row_off[i];
    int64_t z0 = row_ptr[g0], m = row_ptr[g0 + n] - z0;
    trip_t* t = (trip_t*)malloc(sizeof(trip_t) * (size_t)(m > 0 ? m : 1));
    for (int64_t r = 0; r < n; ++r)
      for (int64_t e = row_ptr[g0 + r]; e < row_ptr[g0 + r + 1]; ++e) {
        t[e - z0].row = col[e];        /* transposed: column becomes row */
        t[e - z0].col = (int32_t)r;
        t[e - z0].pos = e - z0;
      }
    qsort(t, (size_t)m, sizeof(trip_t), cmp_trip);
    int64_t e = 0;
    for (int64_t r = 0; r < n; ++r) {
      rowT[g0 + r] = (int32_t)(z0 + e);
      while (e < m && t[e].row == r) ++e;
    }
    for (int64_t g = g0 + n; g < row_off[i + 1]; ++g) rowT[g] = (int32_t)(z0 + m);
    for (int64_t q = 0; q < m; ++q) {
      colT[z0 + q] = t[q].col;
      valsT[z0 + q] = vals[z0 + t[q].pos];
    }
    free(t);
  }
  if (batch > 0) rowT[row_off[batch]] = row_ptr[row_off[batch]];
  return 0;
}

/* O6 SDDMM at the sparsity pattern: out[e] = sum_c D[row_e][c] * B[col_e][c]
 * (fp64 accumulation, one rounding), bound[e] = 1e-5 * sum_c |D||B|. */
int oracle_sddmm(int64_t batch, int32_t k, const int64_t* row_off, const int32_t* sizes,
                 const int32_t* row_ptr, const int32_t* col, const float* B, int64_t ldb,
                 const float* D, int64_t ldd, float* out, double* bound) {
  if (batch < 0 || k < 0) return 1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < batch; ++i) {
    int64_t n = rows_of(row_off, sizes, i);
    for (int64_t r = 0; r < n; ++r) {
      int64_t g = row_off[i] + r;
      for (int64_t e = row_ptr[g]; e < row_ptr[g + 1]; ++e) {
        double acc = 0.0, s = 0.0;
        for (int32_t c = 0; c < k; ++c) {
          double d = (double)D[g * ldd + c];
          double b = (double)B[(row_off[i] + col[e]) * ldb + c];
          acc += d * b;
          s += fabs(d) * fabs(b);
        }
        out[e] = (float)acc;
        if (bound) bound[e] = 1e-5 * s;
      }
    }
  }
  return 0;
}

/* ---- fused GCN layer (NEXT-1): PAPER.md Fig. algo:graph_conv_batched
 * (:304-321) and Eq. (2) (:66-68): for every channel ch,
 *   U_ch = X W_ch,  B_ch = U_ch + 1 bias_ch^T,  C_ch = A_ch B_ch;  Y = sum_ch C_ch.
 * X [N x n_x] (ldx), W [channels][n_x][k] dense, bias [channels][k]; one
 * block-diagonal CSR per channel: row_ptr [channels][N+1] (absolute positions
 * into col / vals), LOCAL column ids.  fp64 throughout, one rounding at the
 * end; mag[g][c] = sum_ch sum_e |a_e| (sum_l |x_{j l}| |w_{l c}| + |b_c|). */
int oracle_gcn_layer(int64_t batch, int32_t channels, int32_t n_x, int32_t k, const int64_t* row_off,
                     const int32_t* row_ptr, const int32_t* col, const float* vals, const float* X,
                     int64_t ldx, const float* W, const float* bias, float* Y, int64_t ldy, double* mag) {
  if (batch < 0 || channels < 1 || n_x < 0 || k < 1) return 1;
  const int64_t N = row_off[batch];
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < batch; ++i) {
    const int64_t n = row_off[i + 1] - row_off[i];
    double* acc = (double*)malloc(sizeof(double) * (size_t)k * 2);
    double* u = (double*)malloc(sizeof(double) * (size_t)k * 2);
    for (int64_t r = 0; r < n; ++r) {
      const int64_t g = row_off[i] + r;
      for (int32_t c = 0; c < k; ++c) acc[c] = 0.0, acc[k + c] = 0.0;
      for (int32_t ch = 0; ch < channels; ++ch) {
        const int32_t* rp = row_ptr + (int64_t)ch * (N + 1);
        const float* Wc = W + (int64_t)ch * n_x * k;
        const float* bc = bias + (int64_t)ch * k;
        for (int64_t e = rp[g]; e < rp[g + 1]; ++e) {
          const int64_t j = row_off[i] + col[e];  /* neighbour's global row */
          const double a = (double)vals[e];
          for (int32_t c = 0; c < k; ++c) {      /* u = X[j] W_ch + bias_ch */
            double s = 0.0, sm = 0.0;
            for (int32_t l = 0; l < n_x; ++l) {
              s += (double)X[j * ldx + l] * (double)Wc[(int64_t)l * k + c];
              sm += fabs((double)X[j * ldx + l]) * fabs((double)Wc[(int64_t)l * k + c]);
            }
            u[c] = s + (double)bc[c];
            u[k + c] = sm + fabs((double)bc[c]);
          }
          for (int32_t c = 0; c < k; ++c) {
            acc[c] += a * u[c];
            acc[k + c] += fabs(a) * u[k + c];
          }
        }
      }
      for (int32_t c = 0; c < k; ++c) {
        Y[g * ldy + c] = (float)acc[c];
        if (mag) mag[g * ldy + c] = acc[k + c];
      }
    }
    free(acc);
    free(u);
  }
  return 0;
}
