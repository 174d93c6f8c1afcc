// Row-tile sparse products fused with the HALS sweep (solver path, sparse A):
//
//   tile_kernel<KP, Src, SWEEP>  one 256-row tile of Y = sum_e a_e T[c_e] per step, computed in
//   shared memory with nnz-balanced slices (a hub row is spread over many lane groups; the first /
//   last row of each slice goes to a carry slot, carries combined in slice order: no atomics), then
//     SWEEP = false: Yout[tile] = Yin[tile] + y            (a partial product over a column block)
//     SWEEP = true : b = Yin[tile] + y + alpha F[tile]; the HALS sweep of each row (Eq. 2.6,
//                    P:170-175) with G (+alpha I); X written; the updated rows accumulated into
//                    X^T X (P:420 / P:690) and, in the last CTA, its Cholesky factor.
//
// Sources (what "entry e of row r" is):
//   CsrSrc     nonzeros [lo[r], hi[r]) of CSR A with gather table T = F: the exact product A F
//              (P:181).  With column cuts (lo/hi = the first nonzero of row r at or
//              after a column boundary; columns are sorted within a row) a pass covers one column
//              block of A, so the rows of F it gathers (n/NB x 128 B) stay resident in L2; the
//              partial products of the blocks are summed through Yin / Yout.
//   BucketSrc  entries [off[r], off[r+1]) of the destination buckets of the sampled rows (bucket.cu)
//              with gather table T = Z, Z[t] = omega_t f_{u_t}: the sampled product
//              Y_s = sum_{i in U} omega_i A[i,:]^T f_i (reading Z28).
#include "fused_common.cuh"

namespace symnmf {

constexpr int kTR = 256;         // rows per tile = threads per CTA
constexpr int kTUE = 8;          // gathers in flight per lane group

struct CsrSrc {
  const int64_t* lo;
  const int64_t* hi;
  const int32_t* col;
  const float* val;
  __device__ __forceinline__ int64_t lo_of(int64_t r) const { return lo[r]; }
  __device__ __forceinline__ int64_t hi_of(int64_t r) const { return hi[r]; }
  __device__ __forceinline__ void load(int64_t e, int& c, float& a) const {
    c = __ldcs(col + e);
    a = __ldcs(val + e);
  }
};

struct BucketSrc {
  const int32_t* off;
  const int2* ent;
  __device__ __forceinline__ int64_t lo_of(int64_t r) const { return off[r]; }
  __device__ __forceinline__ int64_t hi_of(int64_t r) const { return off[r + 1]; }
  __device__ __forceinline__ void load(int64_t e, int& c, float& a) const {
    const int2 x = __ldcs(ent + e);
    c = x.x;
    a = __int_as_float(x.y);
  }
};

template <class Src>
struct TileArgs {
  Src src;
  int64_t n;
  const float4* T;        // gather table, rows of KP floats
  const float* Yin;       // nullable: partial product added to the tile (n x KP)
  float* Yout;            // !SWEEP: output partial product (n x KP)
  // SWEEP only
  const float* F;         // alpha term rows (the fixed factor)
  const double* G;
  double alpha;
  float* X;
  double* Gacc;
  double* Gout;
  float* Rf32;
  unsigned int* counter;
  int32_t* status;
};

__device__ __forceinline__ int tile_row_of2(const int* sOff, int rows, int e) {   // sOff[r] <= e < sOff[r+1]
  int lo = 0, hi = rows - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (sOff[mid] <= e) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Per-thread upper 4x4 block (ai <= bi) of the tile Gram: fp32 over one tile, added into this
// thread's fp64 slot in shared memory; committed once per CTA (fixed order) into a replica.
template <int KP>
struct TileGram {
  static constexpr int NB = KP / 4, PAIRS = NB * (NB + 1) / 2;
  int ai, bi, g, RG, p;
  bool active;
  __device__ void init(int t) {
    RG = kTR / PAIRS;
    g = t / PAIRS;
    p = t - g * PAIRS;
    active = g < RG;
    int a = 0, rem = p;
    while (rem >= NB - a) { rem -= NB - a; ++a; }
    ai = a; bi = a + rem;
  }
  __device__ void tile(const float* s, int stride, int rows, double* slot) const {
    if (!active) return;
    float acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.f;
    for (int r = g; r < rows; r += RG) {
      const float4 a4 = *reinterpret_cast<const float4*>(s + r * stride + 4 * ai);
      const float4 b4 = *reinterpret_cast<const float4*>(s + r * stride + 4 * bi);
      const float a[4] = {a4.x, a4.y, a4.z, a4.w}, b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i * 4 + j] = fmaf(a[i], b[j], acc[i * 4 + j]);
    }
    double* my = slot + (size_t)threadIdx.x * 16;
#pragma unroll
    for (int e = 0; e < 16; ++e) my[e] += (double)acc[e];
  }
  __device__ void commit(const double* slot, double* Gacc) const {
    __syncthreads();
    double* rep = Gacc + (size_t)(blockIdx.x % kGramReplicas) * KP * KP;
    for (int idx = threadIdx.x; idx < PAIRS * 16; idx += kTR) {
      const int pp = idx >> 4, e = idx & 15;
      double sum = 0.0;
      for (int gg = 0; gg < kTR / PAIRS; ++gg) sum += slot[(size_t)(gg * PAIRS + pp) * 16 + e];
      int a0 = 0, rem = pp;
      while (rem >= NB - a0) { rem -= NB - a0; ++a0; }
      const int a = 4 * a0 + (e >> 2), b = 4 * (a0 + rem) + (e & 3);
      if (a <= b && sum != 0.0) atomicAdd(rep + a * KP + b, sum);
    }
  }
};

template <int KP>
struct TileLayout {
  static constexpr int ST = KP + 4;
  static constexpr int NSLICE = (kTR / 32) * (32 / (KP / 4));   // lane groups
  static constexpr int NCARRY = 2 * NSLICE;
  static constexpr size_t y = 0;                                                 // float [TR][ST]
  static constexpr size_t carry = y + sizeof(float) * kTR * ST;                  // float [NCARRY][KP]
  static constexpr size_t crow = carry + sizeof(float) * NCARRY * KP;            // int [NCARRY]
  static constexpr size_t base = crow + sizeof(int) * NCARRY;                    // int64 [TR]: lo(r) - sOff[r]
  static constexpr size_t gram = (base + sizeof(int64_t) * kTR + 15) & ~size_t(15);   // double [TR][16]
  static constexpr size_t bytes_partial = gram;
  static constexpr size_t bytes_sweep = gram + sizeof(double) * kTR * 16;
};

template <int KP, class Src, bool SWEEP>
__global__ void __launch_bounds__(kTR, 2) tile_kernel(const TileArgs<Src> a) {
  using L = TileLayout<KP>;
  constexpr int ST = L::ST, LPR = KP / 4, NG = 32 / LPR;
  __shared__ __align__(16) float sG[SWEEP ? KP * KP : 4];   // sG[i*KP + j] = G[j][i], 0 on the diagonal
  __shared__ float sInv[SWEEP ? KP : 1];
  __shared__ int sOk[SWEEP ? KP : 1];
  __shared__ int sOff[kTR + 1];
  __shared__ int sScan[33];
  extern __shared__ __align__(16) unsigned char smt[];
  float* sY = reinterpret_cast<float*>(smt + L::y);
  float* sC = reinterpret_cast<float*>(smt + L::carry);
  int* sCr = reinterpret_cast<int*>(smt + L::crow);
  int64_t* sBase = reinterpret_cast<int64_t*>(smt + L::base);
  if (dev_failed(a.status)) return;
  const int64_t n = a.n;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, grp = lane / LPR, li = lane % LPR;
  double* gslot = reinterpret_cast<double*>(smt + L::gram);
  TileGram<KP> gt;
  float a32 = 0.f;
  if constexpr (SWEEP) {
    for (int e = tid; e < KP * KP; e += kTR) {
      const int i = e / KP, j = e - i * KP;
      sG[e] = (i != j) ? (float)a.G[j * KP + i] : 0.f;
    }
    for (int i = tid; i < KP; i += kTR) {
      const double den = a.G[i * KP + i] + a.alpha;
      sOk[i] = den > 0.0;
      sInv[i] = den > 0.0 ? (float)(1.0 / den) : 0.f;
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) gslot[tid * 16 + e] = 0.0;
    gt.init(tid);
    a32 = (float)a.alpha;
  }
  const int64_t tiles = (n + kTR - 1) / kTR;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t r0 = t * kTR;
    const int rows = (int)min64(kTR, n - r0);
    if constexpr (SWEEP) {
      if (tid < rows) {   // the sweep's X and F rows: fetched into L2 while the product runs
#pragma unroll
        for (int c = 0; c < KP; c += 32) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a.X + (r0 + tid) * KP + c));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a.F + (r0 + tid) * KP + c));
        }
      }
    }
    // entry ranges of the tile's rows -> exclusive offsets in the tile
    int64_t lo = 0;
    int len = 0;
    if (tid < rows) {
      lo = a.src.lo_of(r0 + tid);
      len = (int)(a.src.hi_of(r0 + tid) - lo);
    }
    __syncthreads();   // previous tile's reads of sY / sOff are done
    int tot;
    const int ex = block_excl_scan(len, sScan, &tot);
    sOff[tid] = ex;
    sBase[tid] = lo - ex;
    if (tid == 0) sOff[kTR] = tot;
    for (int e = tid; e < L::NCARRY * KP; e += kTR) sC[e] = 0.f;
    if (tid < L::NCARRY) sCr[tid] = -1;
    if (a.Yin) {   // coalesced: the tile's partial-product rows are contiguous
      const float4* Yt = reinterpret_cast<const float4*>(a.Yin) + r0 * LPR;
      for (int q = tid; q < rows * LPR; q += kTR) {
        const int r = q / LPR, c = q - r * LPR;
        *reinterpret_cast<float4*>(sY + r * ST + 4 * c) = __ldcs(Yt + q);
      }
    } else {
#pragma unroll
      for (int c = 0; c < KP; c += 4)
        *reinterpret_cast<float4*>(sY + tid * ST + c) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    const int total = tot;
    {
      // ---- nnz-balanced slices, one per lane group; interior rows added, first / last carried
      const int sl = wid * NG + grp;
      const int Ls = (total + L::NSLICE - 1) / L::NSLICE;
      const int s0 = min(total, sl * Ls), s1 = min(total, s0 + Ls);
      if (s0 < s1) {
        const int rfirst = tile_row_of2(sOff, rows, s0), rlast = tile_row_of2(sOff, rows, s1 - 1);
        int row = rfirst;                                   // row being accumulated
        int lrow = rfirst, lrend = sOff[rfirst + 1];        // row of the entries being loaded
        int64_t leb = sBase[rfirst];
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        auto put = [&](int r, float4 v) {
          if (r == rfirst || r == rlast) {
            float* dst = sC + (2 * sl + (r == rfirst ? 0 : 1)) * KP;
            *reinterpret_cast<float4*>(dst + 4 * li) = v;
          } else {   // interior: this slice owns the row
            float4* d4 = reinterpret_cast<float4*>(sY + r * ST + 4 * li);
            float4 cur = *d4;
            cur.x += v.x; cur.y += v.y; cur.z += v.z; cur.w += v.w;
            *d4 = cur;
          }
        };
        if (li == 0) { sCr[2 * sl] = rfirst; sCr[2 * sl + 1] = rlast != rfirst ? rlast : -1; }
        for (int e = s0; e < s1; e += kTUE) {
          int cc[kTUE], rr[kTUE];
          float aa[kTUE];
          float4 ff[kTUE];
#pragma unroll
          for (int u = 0; u < kTUE; ++u) {
            const int j = e + u;
            if (j < s1) {
              while (j >= lrend) { ++lrow; lrend = sOff[lrow + 1]; leb = sBase[lrow]; }
              rr[u] = lrow;
              a.src.load(leb + j, cc[u], aa[u]);
            } else {
              rr[u] = -1; cc[u] = 0; aa[u] = 0.f;
            }
          }
#pragma unroll
          for (int u = 0; u < kTUE; ++u)
            ff[u] = rr[u] >= 0 ? __ldg(a.T + (int64_t)cc[u] * LPR + li) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int u = 0; u < kTUE; ++u) {
            if (rr[u] >= 0) {
              if (rr[u] != row) {
                put(row, acc);
                acc = make_float4(0.f, 0.f, 0.f, 0.f);
                row = rr[u];
              }
              acc.x = fmaf(aa[u], ff[u].x, acc.x); acc.y = fmaf(aa[u], ff[u].y, acc.y);
              acc.z = fmaf(aa[u], ff[u].z, acc.z); acc.w = fmaf(aa[u], ff[u].w, acc.w);
            }
          }
        }
        put(row, acc);
      }
    }
    __syncthreads();
    // ---- carries: runs of equal rows (consecutive slices) summed in slice order, added once
    for (int e = tid; e < L::NCARRY * LPR; e += kTR) {
      const int c = e / LPR, q = e - c * LPR;
      const int r = sCr[c];
      if (r < 0) continue;
      int prev = c - 1;
      while (prev >= 0 && sCr[prev] < 0) --prev;
      if (prev >= 0 && sCr[prev] == r) continue;   // not the head of its run
      float4 s = *reinterpret_cast<const float4*>(sC + c * KP + 4 * q);
      for (int c2 = c + 1; c2 < L::NCARRY; ++c2) {
        const int r2 = sCr[c2];
        if (r2 < 0) continue;
        if (r2 != r) break;
        const float4 v = *reinterpret_cast<const float4*>(sC + c2 * KP + 4 * q);
        s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
      }
      float4* d4 = reinterpret_cast<float4*>(sY + r * ST + 4 * q);
      float4 cur = *d4;
      cur.x += s.x; cur.y += s.y; cur.z += s.z; cur.w += s.w;
      *d4 = cur;
    }
    __syncthreads();
    if constexpr (!SWEEP) {
      float4* Yt = reinterpret_cast<float4*>(a.Yout) + r0 * LPR;
      for (int q = tid; q < rows * LPR; q += kTR) {
        const int r = q / LPR, c = q - r * LPR;
        __stcs(Yt + q, *reinterpret_cast<const float4*>(sY + r * ST + 4 * c));
      }
    } else {
      // ---- b = y + alpha f for the tile (coalesced: the tile's F rows are contiguous)
      {
        const float4* Ft = reinterpret_cast<const float4*>(a.F) + r0 * LPR;
        for (int q = tid; q < rows * LPR; q += kTR) {
          const int r = q / LPR, c = q - r * LPR;
          const float4 fv = __ldg(Ft + q);
          float4* d4 = reinterpret_cast<float4*>(sY + r * ST + 4 * c);
          float4 y = *d4;
          y.x = fmaf(a32, fv.x, y.x); y.y = fmaf(a32, fv.y, y.y); y.z = fmaf(a32, fv.z, y.z); y.w = fmaf(a32, fv.w, y.w);
          *d4 = y;
        }
      }
      __syncthreads();
      // ---- HALS sweep of row tid, Gauss-Seidel over the KP columns (x in registers, b in smem)
      if (tid < rows) {
        const int64_t r = r0 + tid;
        float x[KP];
        const float4* X4 = reinterpret_cast<const float4*>(a.X + r * KP);
#pragma unroll
        for (int j = 0; j < KP; j += 4) {
          const float4 xv = X4[j / 4];
          x[j] = xv.x; x[j + 1] = xv.y; x[j + 2] = xv.z; x[j + 3] = xv.w;
        }
        const float* brow = sY + tid * ST;
#pragma unroll
        for (int i = 0; i < KP; ++i) {
          float s0 = brow[i], s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
          for (int j = 0; j < KP; j += 4) {
            const float4 g = *reinterpret_cast<const float4*>(sG + i * KP + j);
            s0 = fmaf(-x[j], g.x, s0);
            s1 = fmaf(-x[j + 1], g.y, s1);
            s2 = fmaf(-x[j + 2], g.z, s2);
            s3 = fmaf(-x[j + 3], g.w, s3);
          }
          const float sv = (s0 + s1) + (s2 + s3);
          if (sOk[i]) x[i] = fmaxf(0.f, sv * sInv[i]);
        }
        float4* Xw = reinterpret_cast<float4*>(a.X + r * KP);
#pragma unroll
        for (int j = 0; j < KP; j += 4) {
          const float4 v = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
          Xw[j / 4] = v;
          *reinterpret_cast<float4*>(sY + tid * ST + j) = v;
        }
      }
      __syncthreads();
      gt.tile(sY, ST, rows, gslot);
    }
  }
  if constexpr (SWEEP) {
    // ---- commit the CTA's X^T X into a replica of the global accumulator; last CTA finalizes
    gt.commit(gslot, a.Gacc);
    if (arrive_last(a.counter)) {
      double* sa = reinterpret_cast<double*>(smt);
      finalize_gram<KP>(a.Gacc, a.Gout, KP, a.Rf32, sa, sa + KP * (KP + 1), a.status);
    }
  }
}

template <int KP, class Src, bool SWEEP>
static void tile_launch(const TileArgs<Src>& a, cudaStream_t st) {
  using L = TileLayout<KP>;
  size_t smem = SWEEP ? std::max({L::bytes_sweep, sizeof(double) * 2 * KP * (KP + 1), size_t(32768)})
                      : L::bytes_partial;
  const int64_t tiles = (a.n + kTR - 1) / kTR;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 148 * 2));
  cudaFuncSetAttribute(tile_kernel<KP, Src, SWEEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_pdl(tile_kernel<KP, Src, SWEEP>, grid, kTR, smem, st, a);
}

template <class Src, bool SWEEP>
static void tile_dispatch(int k, const TileArgs<Src>& a, cudaStream_t st) {
  switch (k) {
    case 8: tile_launch<8, Src, SWEEP>(a, st); break;
    case 16: tile_launch<16, Src, SWEEP>(a, st); break;
    case 32: tile_launch<32, Src, SWEEP>(a, st); break;
    default: tile_launch<64, Src, SWEEP>(a, st); break;
  }
}

// Exact CSR product in column-block passes (nb >= 1, cuts = (nb - 1) x n first-nonzero indices),
// the last fused with the sweep; Ypart (n x k) carries the partial sums between passes.
void launch_csr_tile_passes(const symnmf_matrix& A, int nb, const int64_t* cuts, float* Ypart, const float* F,
                            const double* G, double alpha, float* X, int64_t n, int k, double* Gacc, double* Gout,
                            float* Rf32, unsigned int* counter, int32_t* status, cudaStream_t st) {
  for (int b = 0; b < nb; ++b) {
    TileArgs<CsrSrc> a{};
    a.src.lo = b == 0 ? A.rowptr : cuts + (size_t)(b - 1) * n;
    a.src.hi = b == nb - 1 ? A.rowptr + 1 : cuts + (size_t)b * n;
    a.src.col = A.colidx;
    a.src.val = A.val;
    a.n = n;
    a.T = reinterpret_cast<const float4*>(F);
    a.Yin = b == 0 ? nullptr : Ypart;
    a.status = status;
    if (b < nb - 1) {
      a.Yout = Ypart;
      tile_dispatch<CsrSrc, false>(k, a, st);
    } else {
      a.F = F; a.G = G; a.alpha = alpha; a.X = X; a.Gacc = Gacc; a.Gout = Gout; a.Rf32 = Rf32; a.counter = counter;
      tile_dispatch<CsrSrc, true>(k, a, st);
    }
  }
}

// Sampled product from the destination buckets, fused with the sweep.
void launch_bucket_tile_sweep(const BucketWs& b, const float* Z, const float* F, const double* G, double alpha,
                              float* X, int64_t n, int k, double* Gacc, double* Gout, float* Rf32,
                              unsigned int* counter, int32_t* status, cudaStream_t st) {
  TileArgs<BucketSrc> a{};
  a.src.off = b.off;
  a.src.ent = b.ent;
  a.n = n;
  a.T = reinterpret_cast<const float4*>(Z);
  a.F = F; a.G = G; a.alpha = alpha; a.X = X; a.Gacc = Gacc; a.Gout = Gout; a.Rf32 = Rf32; a.counter = counter;
  a.status = status;
  tile_dispatch<BucketSrc, true>(k, a, st);
}

// ---------------------------------------------------------------- column cuts (setup, once per A)
// cuts[(b - 1) n + r] = first nonzero of row r with column >= b n / nb, b = 1..nb-1 (binary search of
// the sorted row); also validates that every row's columns are sorted, unique and in [0, n).
__global__ void csr_cuts_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col, int64_t n,
                                int nb, int64_t* __restrict__ cuts, int32_t* __restrict__ bad) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t e0 = rowptr[r], e1 = rowptr[r + 1];
  for (int64_t e = e0; e < e1; ++e) {
    const int32_t c = col[e];
    if (c < 0 || c >= n || (e > e0 && c <= col[e - 1])) { atomicExch(bad, 1); break; }
  }
  for (int b = 1; b < nb; ++b) {
    const int64_t cb = n * b / nb;
    int64_t lo = e0, hi = e1;
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if (col[m] < cb) lo = m + 1; else hi = m;
    }
    cuts[(size_t)(b - 1) * n + r] = lo;
  }
}

void launch_csr_cuts(const symnmf_matrix& A, int nb, int64_t* cuts, int32_t* bad, cudaStream_t st) {
  csr_cuts_kernel<<<(unsigned)((A.n + 255) / 256), 256, 0, st>>>(A.rowptr, A.colidx, A.n, nb, cuts, bad);
}

}  // namespace symnmf
