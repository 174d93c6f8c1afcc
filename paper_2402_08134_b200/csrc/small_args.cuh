// Arguments of the persistent small-problem LvS iteration kernel (small.cu), filled by the
// solver (api.cu).  All pointers are device pointers into the solver's workspace or the
// caller's buffers.
#pragma once
#include "kernels.cuh"

namespace symnmf {

struct SmallArgs {
  int32_t kind;
  int64_t n, lda;
  const float* val;
  const int64_t* rowptr;
  const int32_t* colidx;
  float* W;
  float* H;
  int k;
  double alpha, T;
  int64_t s;
  uint64_t seed;
  int32_t* iter_dev;
  int32_t first_iter, max_iters;
  symnmf_half_stats* stats;
  float* lev;
  uint64_t* bw;
  uint32_t* bd;
  double* bt;
  uint32_t* bu;
  uint64_t* P;
  int32_t* cnt;
  symnmf_plan plan;
  float* Y;              // n x k; zero between halves when A is CSR (scatter target)
  double* GsAcc;         // kGramReplicas x k x k, zero on entry
  double* GAcc;          // kGramReplicas x k x k, zero on entry
  double* Gout;          // k x k: X^T X of the last half (H^T H at the end of an iteration)
  float* R32;            // KP x KP upper R | 1 / diag(R): CholeskyQR factor of H^T H (in and out)
  unsigned int* bar;     // [count, generation] of the grid barrier
  int32_t* status;
};

}  // namespace symnmf
