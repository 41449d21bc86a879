// partition.cpp — multi-GPU batch partitioner (hot-path row a-7).
//
// The paper is single-GPU ("we used only one GPU"); north_star
// asks for graphs sharded across the GPUs of one box, balanced by nnz*k, with
// no collective on the hot path.  Graphs are independent (C is block
// diagonal), so a contiguous split needs no exchange.  Rule (R25):
// cost c_i = nnz_i * k, prefix P_j, total T; split[r] = smallest j with
// P_j * parts >= r * T, found with one forward sweep (j is monotone in r).
// Integer-only (128-bit products), so every rank computes the same split.
#include "internal.h"

extern "C" BSPMM_API bspmm_status_t bspmm_partition(int32_t batch, const int64_t* nnz_off, int32_t k,
                                                    int32_t parts, int32_t* split) {
  if (batch < 0 || k < 0 || parts < 1 || !split || (batch > 0 && !nnz_off)) return BSPMM_ERROR_INVALID_VALUE;
  split[0] = 0;
  split[parts] = batch;
  if (batch == 0) {
    for (int32_t r = 1; r < parts; ++r) split[r] = 0;
    return BSPMM_SUCCESS;
  }
  const int64_t base = nnz_off[0];
  for (int32_t i = 0; i < batch; ++i)
    if (nnz_off[i + 1] < nnz_off[i]) return BSPMM_ERROR_INVALID_VALUE;
  const __int128 T = (__int128)(nnz_off[batch] - base) * k;
  if (T == 0) {
    for (int32_t r = 1; r < parts; ++r) split[r] = (int32_t)((int64_t)r * batch / parts);
    return BSPMM_SUCCESS;
  }
  int64_t j = 0;
  for (int32_t r = 1; r < parts; ++r) {
    const __int128 need = (__int128)r * T;
    while (j < batch && (__int128)(nnz_off[j] - base) * k * parts < need) ++j;
    split[r] = (int32_t)j;
  }
  return BSPMM_SUCCESS;
}
