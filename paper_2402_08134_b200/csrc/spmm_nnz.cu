// (a10) The exact CSR product Y = A F, balanced by
// nonzeros: the nnz range is cut into equal chunks of kChunk nonzeros, one per group of k/4 lanes
// (float4 per lane), so a hub row is spread over many groups and every group gathers the same
// number of rows of F.  Rows complete inside a chunk are stored by its group; the partial sums of
// the (at most two) rows a chunk shares with its neighbours go to carry slots, and spmm_nnz_fix
// sums them in chunk order (deterministic, no atomics) and writes the empty rows.  The first row of
// each chunk is found once per A (spmm_nnz_rows, at solver creation).
#include "kernels.cuh"

namespace symnmf {

constexpr int kChunk = 256;        // nonzeros per lane group
constexpr int kGather = 8;         // rows of F in flight per lane group

int64_t spmm_nnz_chunks(int64_t nnz) { return (nnz + kChunk - 1) / kChunk; }

struct NnzCsr {      // CSR A: rowptr int64, separate col / val
  const int64_t* rowptr;
  const int32_t* col;
  const float* val;
  __device__ __forceinline__ int64_t ptr(int64_t r) const { return rowptr[r]; }
  __device__ __forceinline__ void load(int64_t e, int& c, float& a) const {
    c = __ldcs(col + e);
    a = __ldcs(val + e);
  }
};
// chunk_row[g] = the row holding entry g * kChunk (largest r with ptr(r) <= g * kChunk), for the
// chunks of `total` entries (*total_dev when given)
template <class Src>
__global__ void spmm_nnz_rows_kernel(Src src, int64_t n, int64_t total, const int32_t* __restrict__ total_dev,
                                     int64_t* __restrict__ chunk_row, const int32_t* __restrict__ status) {
  if (status && dev_failed(status)) return;
  const int64_t nnz = total_dev ? (int64_t)*total_dev : total;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g * kChunk >= nnz) return;
  const int64_t s0 = g * kChunk;
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (src.ptr(mid) <= s0) lo = mid; else hi = mid - 1;
  }
  chunk_row[g] = lo;
}

template <int KP, class Src>
__global__ void __launch_bounds__(256, 3) spmm_nnz(Src src, int64_t total, const int32_t* __restrict__ total_dev,
                                                   const int64_t* __restrict__ chunk_row,
                                                   const float4* __restrict__ F4, float4* __restrict__ Y4,
                                                   float4* __restrict__ carry, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  constexpr int LPR = KP / 4;                        // lanes per group (float4 each)
  constexpr int LG = LPR < kGather ? LPR : kGather;  // lanes that load a batch's entries
  constexpr int PER = kGather / LG;                  // entries each loading lane holds
  const int lane = threadIdx.x & 31, li = lane % LPR;
  const unsigned gmask = (LPR == 32 ? 0xffffffffu : ((1u << LPR) - 1u) << (lane - li));
  const int64_t nnz = total_dev ? (int64_t)*total_dev : total;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / LPR;
  const int64_t nchunks = (nnz + kChunk - 1) / kChunk;
  for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPR; g < nchunks; g += ng) {
    const int64_t s0 = g * kChunk, s1 = min64(nnz, s0 + kChunk);
    const int64_t rf = chunk_row[g];
    int64_t r = rf;
    int64_t rstart = src.ptr(r), rend = src.ptr(r + 1);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    auto emit = [&]() {
      if (rstart >= s0 && rend <= s1) Y4[r * LPR + li] = acc;                 // complete in this chunk
      else carry[(2 * g + (r == rf ? 0 : 1)) * LPR + li] = acc;               // shared with a neighbour
    };
    // the batch's entries: lane li < LG loads entries e + li + LG p (coalesced), shared by shuffles;
    // the next batch's are loaded before this batch's gathers, so the entry stream's latency
    // overlaps the gathers' (ncu r2: the two dependent loads per batch were the top two stalls)
    int cm[PER];
    float am[PER];
    auto load_batch = [&](int64_t e) {
#pragma unroll
      for (int p = 0; p < PER; ++p) {
        const int64_t ej = e + li + LG * p;
        if (li < LG && ej < s1) src.load(ej, cm[p], am[p]); else { cm[p] = 0; am[p] = 0.f; }
      }
    };
    load_batch(s0);
    for (int64_t e = s0; e < s1; e += kGather) {
      int cc[kGather];
      float aa[kGather];
#pragma unroll
      for (int u = 0; u < kGather; ++u) {
        cc[u] = __shfl_sync(gmask, cm[u / LG], u % LG, LPR);
        aa[u] = __shfl_sync(gmask, am[u / LG], u % LG, LPR);
      }
      load_batch(e + kGather);
      float4 ff[kGather];
#pragma unroll
      for (int u = 0; u < kGather; ++u)
        ff[u] = (e + u < s1) ? __ldg(F4 + (int64_t)cc[u] * LPR + li) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < kGather; ++u) {
        const int64_t ei = e + u;
        if (ei < s1) {
          if (ei >= rend) {                 // row r ends: store it, move to the row holding ei
            emit();
            acc = make_float4(0.f, 0.f, 0.f, 0.f);
            do { ++r; rstart = rend; rend = src.ptr(r + 1); } while (rend <= ei);   // skips empty rows
          }
          acc.x = fmaf(aa[u], ff[u].x, acc.x); acc.y = fmaf(aa[u], ff[u].y, acc.y);
          acc.z = fmaf(aa[u], ff[u].z, acc.z); acc.w = fmaf(aa[u], ff[u].w, acc.w);
        }
      }
    }
    emit();
  }
}

// Rows shared between chunks: the carries of every chunk they touch, in chunk order; empty rows: 0.
template <int KP, class Src>
__global__ void __launch_bounds__(256) spmm_nnz_fix(Src src, int64_t n, const float4* __restrict__ carry,
                                                    float4* __restrict__ Y4, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  constexpr int LPR = KP / 4;
  const int li = threadIdx.x % LPR;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / LPR;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPR; r < n; r += ng) {
    const int64_t a = src.ptr(r), b = src.ptr(r + 1);
    if (a == b) { Y4[r * LPR + li] = make_float4(0.f, 0.f, 0.f, 0.f); continue; }
    const int64_t c0 = a / kChunk, c1 = (b - 1) / kChunk;
    if (c0 == c1) continue;                                      // stored by its chunk
    // in c0 the row is the chunk's first row iff it starts at the chunk start, else its last row
    float4 s = carry[(2 * c0 + (a == c0 * kChunk ? 0 : 1)) * LPR + li];
    for (int64_t c = c0 + 1; c <= c1; ++c) {
      const float4 v = carry[(2 * c) * LPR + li];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    Y4[r * LPR + li] = s;
  }
}

size_t spmm_nnz_carry_floats(int64_t nnz, int k) { return (size_t)2 * spmm_nnz_chunks(nnz) * k; }

void launch_spmm_nnz_rows(const symnmf_matrix& A, int64_t* chunk_row, cudaStream_t st) {
  const int64_t nc = spmm_nnz_chunks(A.nnz);
  if (nc > 0)
    spmm_nnz_rows_kernel<NnzCsr><<<(unsigned)((nc + 255) / 256), 256, 0, st>>>(
        NnzCsr{A.rowptr, A.colidx, A.val}, A.n, A.nnz, nullptr, chunk_row, nullptr);
}

template <int KP, class Src>
static void spmm_nnz_t(Src src, int64_t n, int64_t total_cap, const int32_t* total_dev, const int64_t* chunk_row,
                       const float* F, float* Y, float* carry, const int32_t* status, cudaStream_t st) {
  constexpr int LPR = KP / 4;
  const int64_t groups = spmm_nnz_chunks(total_cap);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((groups * LPR + 255) / 256, 148 * 16));
  if (total_cap > 0)
    launch_pdl(spmm_nnz<KP, Src>, grid, 256, 0, st, src, total_cap, total_dev, chunk_row,
               reinterpret_cast<const float4*>(F), reinterpret_cast<float4*>(Y), reinterpret_cast<float4*>(carry),
               status);
  const int gridf = (int)std::max<int64_t>(1, std::min<int64_t>((n * LPR + 255) / 256, 148 * 16));
  launch_pdl(spmm_nnz_fix<KP, Src>, gridf, 256, 0, st, src, n, reinterpret_cast<const float4*>(carry),
             reinterpret_cast<float4*>(Y), status);
}

template <class Src>
static void spmm_nnz_k(Src src, int64_t n, int64_t total_cap, const int32_t* total_dev, const int64_t* chunk_row,
                       const float* F, int k, float* Y, float* carry, const int32_t* status, cudaStream_t st) {
  switch (k) {
    case 8: spmm_nnz_t<8>(src, n, total_cap, total_dev, chunk_row, F, Y, carry, status, st); break;
    case 16: spmm_nnz_t<16>(src, n, total_cap, total_dev, chunk_row, F, Y, carry, status, st); break;
    case 32: spmm_nnz_t<32>(src, n, total_cap, total_dev, chunk_row, F, Y, carry, status, st); break;
    default: spmm_nnz_t<64>(src, n, total_cap, total_dev, chunk_row, F, Y, carry, status, st); break;
  }
}

bool spmm_nnz_supported(int k) { return k == 8 || k == 16 || k == 32 || k == 64; }

void launch_spmm_nnz(const symnmf_matrix& A, const int64_t* chunk_row, const float* F, int k, float* Y, float* carry,
                     const int32_t* status, cudaStream_t st) {
  spmm_nnz_k(NnzCsr{A.rowptr, A.colidx, A.val}, A.n, A.nnz, nullptr, chunk_row, F, k, Y, carry, status, st);
}

// ---------------------------------------------------------------- CSR input check (once per A)
// *bad = 1 if some row's column indices are not sorted, unique and in [0, n) (caller zeroes *bad).
__global__ void csr_check_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col, int64_t n,
                                 int32_t* __restrict__ bad) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= n) return;
  const int lane = threadIdx.x & 31;
  const int64_t e0 = rowptr[r], e1 = rowptr[r + 1];
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    const int32_t c = col[e];
    if (c < 0 || c >= n || (e > e0 && c <= col[e - 1])) atomicExch(bad, 1);
  }
}

void launch_csr_check(const symnmf_matrix& A, int32_t* bad, cudaStream_t st) {
  if (A.n > 0) csr_check_kernel<<<(unsigned)((A.n + 7) / 8), 256, 0, st>>>(A.rowptr, A.colidx, A.n, bad);
}

}  // namespace symnmf
