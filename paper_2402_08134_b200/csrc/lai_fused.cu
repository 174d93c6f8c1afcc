// (a13) + (a11) fused: one LAI-SymNMF half (Alg. LAI-SymNMF) in one launch.
//
// The half needs Y = U (Lambda (U^T F)) and the sweep of X against
// (F^T F + alpha I, Y + alpha F) (Eq. 2.6).  U^T F is a reduction over
// all n rows, so it is produced by the PREVIOUS half's launch, where F was that half's
// output X: each launch, besides the sweep, accumulates X^T X (the next half's Gram) and
// U^T X (the next half's l x k product), and its last CTA forms G_next = X^T X and
// M_next = Lambda U^T X (fp32).  Per 128-row tile:
//   1. U tile (128 x l) -> shared memory; Y = U M by 8 x 4 register blocks (M = Lambda U^T F in smem)
//   2. b = Y + alpha F (coalesced F tile), sweep of row r by thread r (x in registers), X written
//   3. X^T X (upper 4x4 blocks) and U^T X (4x4 blocks) over the tile: fp32 per tile, fp64
//      registers across tiles, fp64 red.add per CTA into replicas, last CTA finalizes.
#include "fused_common.cuh"

namespace symnmf {

constexpr int LT = 256;    // threads
constexpr int LTR = 128;   // rows per tile

template <int KP, int LP>   // factor width, padded sketch width (LP % 4 == 0, l <= LP)
struct LaiSmem {
  static constexpr int US = LP + 4, XS = KP + 4;
  static constexpr size_t u = 0;                                     // float [LTR][US]
  static constexpr size_t x = u + sizeof(float) * LTR * US;          // float [LTR][XS]   (b, then new x)
  static constexpr size_t m = x + sizeof(float) * LTR * XS;          // float [LP][KP]    M = Lambda U^T F
  static constexpr size_t g = m + sizeof(float) * LP * KP;           // float [KP][KP]    G (transposed, 0 diag)
  static constexpr size_t bytes = g + sizeof(float) * KP * KP;
};

template <int KP, int LP>
__global__ void __launch_bounds__(LT, 1) lai_sweep_fused(const float* __restrict__ U, int l, int64_t n,
                                                         const float* __restrict__ Mcur, const double* __restrict__ G,
                                                         double alpha, const float* __restrict__ F, float* __restrict__ X,
                                                         const double* __restrict__ lam, double* GXacc, double* UXacc,
                                                         double* Gout, float* Mnext, unsigned int* counter,
                                                         int32_t* status) {
  using L = LaiSmem<KP, LP>;
  constexpr int US = L::US, XS = L::XS, Q = KP / 4;
  constexpr int NBX = KP / 4, PX = NBX * (NBX + 1) / 2;   // X^T X upper block pairs
  constexpr int NBU = LP / 4, PU = NBU * NBX;             // U^T X block pairs
  constexpr int PT = PX + PU, PPT = (PT + LT - 1) / LT;
  extern __shared__ __align__(16) unsigned char sml[];
  float* sU = reinterpret_cast<float*>(sml + L::u);
  float* sX = reinterpret_cast<float*>(sml + L::x);
  float* sM = reinterpret_cast<float*>(sml + L::m);
  float* sG = reinterpret_cast<float*>(sml + L::g);
  __shared__ float sInv[KP];
  __shared__ int sOk[KP];
  if (dev_failed(status)) return;
  const int tid = threadIdx.x;
  for (int e = tid; e < LP * KP; e += LT) sM[e] = (e / KP < l) ? Mcur[e] : 0.f;
  for (int e = tid; e < KP * KP; e += LT) {
    const int i = e / KP, j = e - i * KP;
    sG[e] = (i != j) ? -(float)G[j * KP + i] : 0.f;   // negated: the sweep is a chain of FMAs
  }
  for (int i = tid; i < KP; i += LT) {
    const double den = G[i * KP + i] + alpha;
    sOk[i] = den > 0.0;
    sInv[i] = den > 0.0 ? (float)(1.0 / den) : 0.f;
  }
  // block pairs of this thread: p < PX -> (X block ai, X block bi), else (U block ai, X block bi)
  int pa[PPT], pb[PPT];
  bool pu[PPT], pv[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int p = tid + q * LT;
    pv[q] = p < PT;
    pu[q] = p >= PX;
    if (p < PX) {
      int a0 = 0, rem = p;
      while (rem >= NBX - a0) { rem -= NBX - a0; ++a0; }
      pa[q] = a0; pb[q] = a0 + rem;
    } else {
      const int pp = min(p, PT - 1) - PX;
      pa[q] = pp / NBX; pb[q] = pp - pa[q] * NBX;
    }
  }
  double acc64[PPT][16];
#pragma unroll
  for (int q = 0; q < PPT; ++q)
#pragma unroll
    for (int e = 0; e < 16; ++e) acc64[q][e] = 0.0;
  const float a32 = (float)alpha;
  const int rg = tid / 16, cg = tid % 16;   // Y blocks: rows 8 rg .. 8 rg + 7, float4 column chunks cg + 16 cb
  const int64_t tiles = (n + LTR - 1) / LTR;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t r0 = t * LTR;
    const int rows = (int)min64(LTR, n - r0);
    __syncthreads();
    // ---- 1. U tile (rows x l, contiguous) -> sU, zero padded
    {
      const float* Ut = U + r0 * l;
      for (int e = tid; e < rows * l; e += LT) {
        const int r = e / l, a = e - r * l;
        sU[r * US + a] = __ldg(Ut + e);
      }
      for (int e = tid; e < LTR * (US - l); e += LT) {
        const int r = e / (US - l), a = l + e - r * (US - l);
        sU[r * US + a] = 0.f;
      }
      for (int e = tid; e < (LTR - rows) * l; e += LT) {
        const int r = rows + e / l, a = e % l;
        sU[r * US + a] = 0.f;
      }
    }
    __syncthreads();
    // ---- Y = U M (8 x (KP/16 x 4) register block per thread), b = Y + alpha F -> sX
    {
      constexpr int CB = KP / 64;   // float4 column chunks per thread (16 chunk lanes)
      float acc[8][CB * 4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < CB * 4; ++j) acc[i][j] = 0.f;
#pragma unroll 2
      for (int a = 0; a < LP; ++a) {
        float uv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) uv[i] = sU[(8 * rg + i) * US + a];
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
          const float4 m = *reinterpret_cast<const float4*>(sM + a * KP + 4 * (cg + 16 * cb));
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            acc[i][4 * cb] = fmaf(uv[i], m.x, acc[i][4 * cb]);
            acc[i][4 * cb + 1] = fmaf(uv[i], m.y, acc[i][4 * cb + 1]);
            acc[i][4 * cb + 2] = fmaf(uv[i], m.z, acc[i][4 * cb + 2]);
            acc[i][4 * cb + 3] = fmaf(uv[i], m.w, acc[i][4 * cb + 3]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = 8 * rg + i;
        if (r >= rows) continue;
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
          const int c4 = cg + 16 * cb;
          const float4 f = __ldg(reinterpret_cast<const float4*>(F + (r0 + r) * KP) + c4);
          *reinterpret_cast<float4*>(sX + r * XS + 4 * c4) =
              make_float4(fmaf(a32, f.x, acc[i][4 * cb]), fmaf(a32, f.y, acc[i][4 * cb + 1]),
                          fmaf(a32, f.z, acc[i][4 * cb + 2]), fmaf(a32, f.w, acc[i][4 * cb + 3]));
        }
      }
    }
    __syncthreads();
    // ---- sweep of row tid (Gauss-Seidel over the KP columns), b read from sX, x -> sX and X
    if (tid < rows) {
      const int64_t r = r0 + tid;
      float2 x[KP / 2];   // column pairs (packed FFMA2)
      const float4* X4 = reinterpret_cast<const float4*>(X + r * KP);
#pragma unroll
      for (int j = 0; j < KP; j += 4) {
        const float4 v = X4[j / 4];
        x[j / 2] = make_float2(v.x, v.y); x[j / 2 + 1] = make_float2(v.z, v.w);
      }
      const float* brow = sX + tid * XS;
#pragma unroll
      for (int i = 0; i < KP; ++i) {
        float2 s01 = make_float2(brow[i], 0.f), s23 = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < KP; j += 4) {
          const float4 g = *reinterpret_cast<const float4*>(sG + i * KP + j);
          s01 = ffma2(x[j / 2], make_float2(g.x, g.y), s01);
          s23 = ffma2(x[j / 2 + 1], make_float2(g.z, g.w), s23);
        }
        const float sv = (s01.x + s01.y) + (s23.x + s23.y);
        if (sOk[i]) {
          const float v = fmaxf(0.f, sv * sInv[i]);
          if (i & 1) x[i / 2].y = v; else x[i / 2].x = v;
        }
      }
      float4* Xw = reinterpret_cast<float4*>(X + r * KP);
#pragma unroll
      for (int j = 0; j < KP; j += 4) {
        const float4 v = make_float4(x[j / 2].x, x[j / 2].y, x[j / 2 + 1].x, x[j / 2 + 1].y);
        Xw[j / 4] = v;
        *reinterpret_cast<float4*>(sX + tid * XS + j) = v;
      }
    } else if (tid < LTR) {
#pragma unroll
      for (int j = 0; j < KP; j += 4) *reinterpret_cast<float4*>(sX + tid * XS + j) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    // ---- X^T X and U^T X of the tile
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      if (!pv[q]) continue;
      const float* A0 = pu[q] ? sU + 4 * pa[q] : sX + 4 * pa[q];
      const int As = pu[q] ? US : XS;
      float acc[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[e] = 0.f;
      for (int r = 0; r < rows; ++r) {
        const float4 a4 = *reinterpret_cast<const float4*>(A0 + r * As);
        const float4 b4 = *reinterpret_cast<const float4*>(sX + r * XS + 4 * pb[q]);
        const float av[4] = {a4.x, a4.y, a4.z, a4.w}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i * 4 + j] = fmaf(av[i], bv[j], acc[i * 4 + j]);
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) acc64[q][e] += (double)acc[e];
    }
  }
  // ---- commit: fp64 red.add into replica blockIdx % R; the last CTA finalizes
  {
    const int rep = blockIdx.x % kGramReplicas;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      if (!pv[q]) continue;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int i = 4 * pa[q] + (e >> 2), j = 4 * pb[q] + (e & 3);
        if (acc64[q][e] == 0.0) continue;
        if (!pu[q]) {
          if (i <= j) atomicAdd(GXacc + (size_t)rep * KP * KP + i * KP + j, acc64[q][e]);
        } else if (i < l) {
          atomicAdd(UXacc + (size_t)rep * LP * KP + i * KP + j, acc64[q][e]);
        }
      }
    }
  }
  if (!arrive_last(counter)) return;
  for (int e = tid; e < KP * KP; e += LT) {
    const int i = e / KP, j = e - i * KP;
    if (i > j) continue;
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < kGramReplicas; ++r) {
      s += __ldcg(GXacc + (size_t)r * KP * KP + e);
      GXacc[(size_t)r * KP * KP + e] = 0.0;
    }
    Gout[i * KP + j] = s;
    Gout[j * KP + i] = s;
  }
  for (int e = tid; e < LP * KP; e += LT) {
    const int a = e / KP;
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < kGramReplicas; ++r) {
      s += __ldcg(UXacc + (size_t)r * LP * KP + e);
      UXacc[(size_t)r * LP * KP + e] = 0.0;
    }
    if (a < l) Mnext[e] = (float)(lam[a] * s);   // M_next = Lambda U^T X
  }
}

int lai_lp(int l) { return l <= 32 ? 32 : l <= 64 ? 64 : l <= 80 ? 80 : 96; }

bool lai_fused_supported(int k, int l) { return k == 64 && l <= 80; }

template <int KP, int LP>
static void launch_lai_t(const float* U, int l, int64_t n, const float* Mcur, const double* G, double alpha,
                         const float* F, float* X, const double* lam, double* GXacc, double* UXacc, double* Gout,
                         float* Mnext, unsigned int* counter, int32_t* status, cudaStream_t st) {
  const size_t smem = LaiSmem<KP, LP>::bytes;
  cudaFuncSetAttribute(lai_sweep_fused<KP, LP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t tiles = (n + LTR - 1) / LTR;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 148));
  launch_pdl(lai_sweep_fused<KP, LP>, grid, LT, smem, st, U, l, n, Mcur, G, alpha, F, X, lam, GXacc, UXacc, Gout,
             Mnext, counter, status);
}

// Accumulator sizes the caller must provide zeroed: GXacc kGramReplicas x KP x KP, UXacc
// kGramReplicas x LP x KP (left zeroed).  M tables are LP x KP fp32 (rows >= l unused).
void launch_lai_sweep_fused(const float* U, int l, int64_t n, int k, const float* Mcur, const double* G, double alpha,
                            const float* F, float* X, const double* lam, double* GXacc, double* UXacc, double* Gout,
                            float* Mnext, unsigned int* counter, int32_t* status, cudaStream_t st) {
  if (lai_lp(l) <= 64)
    launch_lai_t<64, 64>(U, l, n, Mcur, G, alpha, F, X, lam, GXacc, UXacc, Gout, Mnext, counter, status, st);
  else
    launch_lai_t<64, 80>(U, l, n, Mcur, G, alpha, F, X, lam, GXacc, UXacc, Gout, Mnext, counter, status, st);
  (void)k;
}

}  // namespace symnmf
