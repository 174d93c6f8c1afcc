// (a11) The HALS sweep Update(G + alpha I, Y + alpha F^T) (Eq. 2.6; App. G)
// as a streaming kernel, fused with the Gram of the updated factor (the next half's F^T F, P:420 /
// P:690) and, in the last CTA, its Cholesky factor (CholeskyQR).
//
// sweep_stream<KP>: persistent CTAs of 256 threads, one 256-row tile per step, thread r owning row r.
// The tile's rows of Y, F and X are brought into shared memory with cp.async (16 B chunks, coalesced),
// stored with a padded row stride (k + 4 floats) so that a thread reading its own row and a row group
// reading one row are bank-conflict free; x is held in registers, b = y + alpha f read a chunk at a
// time, and the Gauss-Seidel pass over the k columns takes G (+alpha I) from the constant bank (or
// shared memory).  The new row replaces the old one in the tile, which is then stored coalesced and
// accumulated into the tile Gram (fp32 per tile, fp64 registers across tiles).  Two CTAs per SM:
// one stages its next tile while the other computes.
// Bytes per row: Y, F, X read, X written (+ Y re-zeroed for the scatter paths): 16k (20k) B.
#include <atomic>
#include "fused_common.cuh"

namespace symnmf {

template <int KP>
struct SwL {
  static constexpr int C = KP / 4;              // 16 B chunks per row
  static constexpr int TR = 256;                // rows per tile = threads
  static constexpr int ST = KP + 4;             // padded row stride (floats): a thread reading its own
                                                // row and a row group reading one row are conflict free
  static constexpr size_t arr = sizeof(float) * TR * ST;
  static constexpr size_t y = 0, x = arr, f = 2 * arr;
  static constexpr size_t bytes = 3 * arr;      // Y, X, F staging (X rewritten in place)
  static constexpr size_t bytes_noF = 2 * arr;  // Y carries alpha F: F not staged
  // CTAs per SM the register cap aims at: three when F is not staged (Y carries alpha F: 2 x 37 KB
  // of staging), else two (3 x 110 KB of shared memory do not fit at k = 32)
  static constexpr int per_sm(bool noF) { return noF ? 3 : (KP <= 8 ? 3 : 2); }
};

// Constant-bank copies of the sweep's G (-G_off^T, 1 / (G_ii + alpha), ok flags), one per (solver
// slot, half): with G in the constant bank every FMA of the column loop takes its G operand
// straight from the constant cache (no shared-memory loads, no load-to-use latency).  Written by
// a D2D copy to the symbol (captured in the solver's graph) right before each sweep.
constexpr int kCSlots = 4;
constexpr int kCTab = 32 * 32 + 64;
__constant__ float cSw[2 * kCSlots][kCTab];

template <int KP, int TAB>
struct SwG {   // G source: TAB < 0 -> shared memory, else constant table TAB
  const float* s;
  const float* inv;
  const int* ok;
  __device__ __forceinline__ float4 g4(int i, int j) const {
    if constexpr (TAB < 0) return *reinterpret_cast<const float4*>(s + i * KP + j);
    else return make_float4(cSw[TAB][i * KP + j], cSw[TAB][i * KP + j + 1], cSw[TAB][i * KP + j + 2],
                            cSw[TAB][i * KP + j + 3]);
  }
  __device__ __forceinline__ float invd(int i) const {
    if constexpr (TAB < 0) return inv[i]; else return cSw[TAB][KP * KP + i];
  }
  __device__ __forceinline__ bool okd(int i) const {
    if constexpr (TAB < 0) return ok[i] != 0; else return cSw[TAB][KP * KP + KP + i] != 0.f;
  }
};

template <int KP, int TAB, bool NOF>
__global__ void __launch_bounds__(256, SwL<KP>::per_sm(NOF)) sweep_stream(
    const double* __restrict__ G, double alpha, float* __restrict__ Y, const float* __restrict__ F,
    float* __restrict__ X, int64_t n, int ymode, double* Gacc, double* Gout, float* Rf32, unsigned int* counter,
    int32_t* status) {
  // ymode 0: Y read only; 1: Y re-zeroed for the next scatter; 2: Y holds Y_s + alpha F already (the
  // scatter accumulated onto alpha F), so F is not read, and Y is left as alpha X for the next half,
  // whose fixed factor X is (LvS on CSR: 4nk bytes less per half)
  const bool yalpha = NOF;   // == (ymode == 2)
  using L = SwL<KP>;
  constexpr int C = L::C, TR = L::TR;
  constexpr int NB = KP / 4, PAIRS = NB * (NB + 1) / 2, RG = TR / PAIRS;
  constexpr int ST = L::ST;
  __shared__ __align__(16) float sG[TAB < 0 ? KP * KP : 4];   // sG[i*KP + j] = -G[j][i], 0 on the diagonal
  __shared__ float sInv[KP];
  __shared__ int sOk[KP];
  extern __shared__ __align__(16) unsigned char sms[];
  float* sY = reinterpret_cast<float*>(sms + L::y);
  float* sF = reinterpret_cast<float*>(sms + L::f);
  float* sX = reinterpret_cast<float*>(sms + L::x);
  if (dev_failed(status)) return;
  const int tid = threadIdx.x;
  if constexpr (TAB < 0) {
    for (int e = tid; e < KP * KP; e += TR) {
      const int i = e / KP, j = e - i * KP;
      sG[e] = (i != j) ? -(float)G[j * KP + i] : 0.f;
    }
    for (int i = tid; i < KP; i += TR) {
      const double den = G[i * KP + i] + alpha;
      sOk[i] = den > 0.0;
      sInv[i] = den > 0.0 ? (float)(1.0 / den) : 0.f;
    }
  }
  // Gram role of this thread: upper 4x4 block (ai, bi) over the rows r = gg (mod RG) of each tile;
  // fp32 over a tile, fp64 registers across tiles
  const int gg = tid / PAIRS, gp = tid - gg * PAIRS;
  int ai = 0, bi = 0;
  {
    int a = 0, rem = gp;
    while (rem >= NB - a) { rem -= NB - a; ++a; }
    ai = a; bi = a + rem;
  }
  const bool gactive = Gacc && gg < RG;
  double acc64[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc64[e] = 0.0;
  const float a32 = (float)alpha;
  const SwG<KP, TAB> gsrc{sG, sInv, sOk};
  const int64_t tiles = (n + TR - 1) / TR;
  __syncthreads();

  // tiles last to first: the product that wrote Y finished with its highest rows, which are the
  // ones still resident in L2; the sweep then ends on the lowest rows, where the next half's
  // leverage / product kernels start
  for (int64_t tt = blockIdx.x; tt < tiles; tt += gridDim.x) {
    const int64_t t = tiles - 1 - tt;
    const int64_t r0 = t * TR;
    const int rows = (int)min64(TR, n - r0);
    // stage the tile's rows of Y, F, X (coalesced 16 B chunks, swizzled)
    for (int q = tid; q < TR * C; q += TR) {
      const int r = q / C, c = q - r * C;
      const bool ok = r < rows;
      const int so = r * ST + 4 * c;
      const int64_t go = ok ? (r0 + r) * KP + 4 * c : 0;
      cp_async16(sY + so, Y + go, ok);
      if (!yalpha) cp_async16(sF + so, F + go, ok);
      cp_async16(sX + so, X + go, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (ymode == 1) {
      float4* Y4 = reinterpret_cast<float4*>(Y) + r0 * C;
      for (int q = tid; q < rows * C; q += TR) __stcs(Y4 + q, make_float4(0.f, 0.f, 0.f, 0.f));
    }
    // x in column pairs: the column loop runs on packed FFMA2 (two FMAs per instruction)
    float2 x2[KP / 2];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const float4 x4 = *reinterpret_cast<const float4*>(sX + tid * ST + 4 * c);
      x2[2 * c] = make_float2(x4.x, x4.y); x2[2 * c + 1] = make_float2(x4.z, x4.w);
    }
    // Gauss-Seidel over the columns of row tid: x_i <- [(b_i - sum_{j != i} G_ij x_j) / (G_ii + alpha)]_+,
    // b = y + alpha f read a 16 B chunk at a time; the table holds -G so every step is an FMA
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int so = tid * ST + 4 * c;
      const float4 y4 = *reinterpret_cast<const float4*>(sY + so);
      const float4 f4 = yalpha ? make_float4(0.f, 0.f, 0.f, 0.f) : *reinterpret_cast<const float4*>(sF + so);
      const float bc[4] = {fmaf(a32, f4.x, y4.x), fmaf(a32, f4.y, y4.y), fmaf(a32, f4.z, y4.z),
                           fmaf(a32, f4.w, y4.w)};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = 4 * c + u;
        float2 s01 = make_float2(bc[u], 0.f), s23 = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < KP; j += 4) {
          const float4 g = gsrc.g4(i, j);
          s01 = ffma2(x2[j / 2], make_float2(g.x, g.y), s01);
          s23 = ffma2(x2[j / 2 + 1], make_float2(g.z, g.w), s23);
        }
        const float sv = (s01.x + s01.y) + (s23.x + s23.y);
        if (gsrc.okd(i)) {
          const float v = fmaxf(0.f, sv * gsrc.invd(i));
          if (i & 1) x2[i / 2].y = v; else x2[i / 2].x = v;
        }
      }
    }
    const bool live = tid < rows;
#pragma unroll
    for (int c = 0; c < C; ++c)   // the new row replaces the old one in the staging tile
      *reinterpret_cast<float4*>(sX + tid * ST + 4 * c) =
          live ? make_float4(x2[2 * c].x, x2[2 * c].y, x2[2 * c + 1].x, x2[2 * c + 1].y)
               : make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    {
      float4* X4 = reinterpret_cast<float4*>(X) + r0 * C;
      float4* Y4 = reinterpret_cast<float4*>(Y) + r0 * C;
      for (int q = tid; q < rows * C; q += TR) {
        const int r = q / C, c = q - r * C;
        const float4 v = *reinterpret_cast<const float4*>(sX + r * ST + 4 * c);
        X4[q] = v;
        if (yalpha) __stcs(Y4 + q, make_float4(a32 * v.x, a32 * v.y, a32 * v.z, a32 * v.w));
      }
    }
    if (gactive) {   // tile Gram of the new rows
      float2 acc[8];   // acc[i * 2 + p] = entries (4 ai + i, 4 bi + 2p .. 2p + 1)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = make_float2(0.f, 0.f);
      const float* pa = sX + gg * ST + 4 * ai;
      const float* pb = sX + gg * ST + 4 * bi;
      int r = gg;
      auto step = [&](int o) {
        const float4 a4 = *reinterpret_cast<const float4*>(pa + o);
        const float4 b4 = *reinterpret_cast<const float4*>(pb + o);
        const float av[4] = {a4.x, a4.y, a4.z, a4.w};
        const float2 b01 = make_float2(b4.x, b4.y), b23 = make_float2(b4.z, b4.w);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[i * 2] = ffma2(make_float2(av[i], av[i]), b01, acc[i * 2]);
          acc[i * 2 + 1] = ffma2(make_float2(av[i], av[i]), b23, acc[i * 2 + 1]);
        }
      };
      for (; r + 3 * RG < rows; r += 4 * RG, pa += 4 * RG * ST, pb += 4 * RG * ST) {
        step(0); step(RG * ST); step(2 * RG * ST); step(3 * RG * ST);
      }
      for (; r < rows; r += RG, pa += RG * ST, pb += RG * ST) step(0);
#pragma unroll
      for (int e = 0; e < 8; ++e) { acc64[2 * e] += (double)acc[e].x; acc64[2 * e + 1] += (double)acc[e].y; }
    }
    __syncthreads();   // staging tile free for the next tile
  }
  if (!Gacc) return;
  // commit: the row groups' partials reduced in shared memory in fixed order, one fp64 red.add per
  // entry into a replica of the global accumulator; the last CTA forms X^T X and its Cholesky factor
  double* red = reinterpret_cast<double*>(sms);       // RG * PAIRS * 16 doubles (<= 32 KB)
  if (gg < RG) {
#pragma unroll
    for (int e = 0; e < 16; ++e) red[(size_t)tid * 16 + e] = acc64[e];
  }
  __syncthreads();
  double* rep = Gacc + (size_t)(blockIdx.x % kGramReplicas) * KP * KP;
  for (int idx = tid; idx < PAIRS * 16; idx += TR) {
    const int pp = idx >> 4, e = idx & 15;
    double sum = 0.0;
    for (int g2 = 0; g2 < RG; ++g2) sum += red[(size_t)(g2 * PAIRS + pp) * 16 + e];
    int a0 = 0, rem = pp;
    while (rem >= NB - a0) { rem -= NB - a0; ++a0; }
    const int a = 4 * a0 + (e >> 2), bb = 4 * (a0 + rem) + (e & 3);
    if (a <= bb && sum != 0.0) atomicAdd(rep + a * KP + bb, sum);
  }
  if (arrive_last(counter)) {
    double* sa = reinterpret_cast<double*>(sms);
    finalize_gram<KP>(Gacc, Gout, KP, Rf32, sa, sa + KP * (KP + 1), status);
  }
}

// fp32 table of the sweep's G for the constant bank: -G_off^T (zero diagonal), 1 / (G_ii + alpha), ok
template <int KP>
__global__ void sweep_table(const double* __restrict__ G, double alpha, float* __restrict__ out,
                            const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  for (int e = threadIdx.x; e < KP * KP; e += blockDim.x) {
    const int i = e / KP, j = e - i * KP;
    out[e] = (i != j) ? -(float)G[j * KP + i] : 0.f;
  }
  for (int i = threadIdx.x; i < KP; i += blockDim.x) {
    const double den = G[i * KP + i] + alpha;
    out[KP * KP + i] = den > 0.0 ? (float)(1.0 / den) : 0.f;
    out[KP * KP + KP + i] = den > 0.0 ? 1.f : 0.f;
  }
}

template <int KP, int TAB>
static void sweep_stream_t(const double* G, double alpha, float* Y, const float* F, float* X, int64_t n, int ymode,
                           double* Gacc, double* Gout, float* Rf32, unsigned int* counter, int32_t* status,
                           cudaStream_t st) {
  using L = SwL<KP>;
  const size_t smem = std::max({ymode == 2 ? L::bytes_noF : L::bytes, sizeof(double) * 2 * KP * (KP + 1),
                                 sizeof(double) * 256 * 16});
  const int64_t tiles = (n + L::TR - 1) / L::TR;
  auto kern = ymode == 2 ? sweep_stream<KP, TAB, true> : sweep_stream<KP, TAB, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, L::TR, smem);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 148 * (int64_t)std::max(1, occ)));
  launch_pdl(kern, grid, L::TR, smem, st, G, alpha, Y, F, X, n, ymode, Gacc, Gout, Rf32, counter, status);
}

bool sweep_stream_supported(int k) { return k == 8 || k == 16 || k == 32; }

// Y = alpha F (the invariant the yalpha sweep keeps for LvS on CSR, set at solver creation)
__global__ void scale_copy_kernel(const float4* __restrict__ F4, float a, float4* __restrict__ Y4, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = F4[i];
    Y4[i] = make_float4(a * v.x, a * v.y, a * v.z, a * v.w);
  }
}
void launch_scale_copy(const float* F, double alpha, float* Y, int64_t count, cudaStream_t st) {
  const int64_t n4 = count / 4;
  if (n4 > 0)
    scale_copy_kernel<<<(unsigned)std::min<int64_t>((n4 + 255) / 256, 148 * 8), 256, 0, st>>>(
        reinterpret_cast<const float4*>(F), (float)alpha, reinterpret_cast<float4*>(Y), n4);
}

// Constant-table slots: a solver takes one for its lifetime (two tables, one per half).
static std::atomic<unsigned> g_cslots{0};
int sweep_cslot_acquire() {
  unsigned m = g_cslots.load();
  for (;;) {
    int b = 0;
    while (b < kCSlots && (m >> b & 1u)) ++b;
    if (b == kCSlots) return -1;
    if (g_cslots.compare_exchange_weak(m, m | (1u << b))) return b;
  }
}
void sweep_cslot_release(int slot) {
  if (slot >= 0) g_cslots.fetch_and(~(1u << slot));
}
size_t sweep_table_floats() { return kCTab; }

template <int KP>
static void sweep_tab_dispatch(int tab, const double* G, double alpha, float* Y, const float* F, float* X, int64_t n,
                               int ymode, double* Gacc, double* Gout, float* Rf32, unsigned int* counter,
                               int32_t* status, cudaStream_t st) {
#define SW_CASE(T) case T: sweep_stream_t<KP, T>(G, alpha, Y, F, X, n, ymode, Gacc, Gout, Rf32, counter, status, st); break;
  switch (tab) {
    SW_CASE(0) SW_CASE(1) SW_CASE(2) SW_CASE(3) SW_CASE(4) SW_CASE(5) SW_CASE(6) SW_CASE(7)
    default: sweep_stream_t<KP, -1>(G, alpha, Y, F, X, n, ymode, Gacc, Gout, Rf32, counter, status, st); break;
  }
#undef SW_CASE
}

// tab >= 0: constant table 2 * slot + side, built from G into `scratch` (sweep_table_floats()) and
// copied to the constant bank first; tab < 0: G staged in shared memory.
void launch_sweep_stream(const double* G, double alpha, float* Y, const float* F, float* X, int64_t n, int k,
                         bool zeroY, double* Gacc, double* Gout, float* Rf32, unsigned int* counter, int32_t* status,
                         cudaStream_t st, int tab, float* scratch, bool yalpha) {
  const int ymode = yalpha ? 2 : zeroY ? 1 : 0;
  if (tab >= 0) {
    const int kp = k;
    switch (kp) {
      case 8: sweep_table<8><<<1, 256, 0, st>>>(G, alpha, scratch, status); break;
      case 16: sweep_table<16><<<1, 256, 0, st>>>(G, alpha, scratch, status); break;
      default: sweep_table<32><<<1, 256, 0, st>>>(G, alpha, scratch, status); break;
    }
    cudaMemcpyToSymbolAsync(cSw, scratch, sizeof(float) * (kp * kp + 2 * kp), sizeof(float) * kCTab * tab,
                            cudaMemcpyDeviceToDevice, st);
  }
  switch (k) {
    case 8: sweep_tab_dispatch<8>(tab, G, alpha, Y, F, X, n, ymode, Gacc, Gout, Rf32, counter, status, st); break;
    case 16: sweep_tab_dispatch<16>(tab, G, alpha, Y, F, X, n, ymode, Gacc, Gout, Rf32, counter, status, st); break;
    default: sweep_tab_dispatch<32>(tab, G, alpha, Y, F, X, n, ymode, Gacc, Gout, Rf32, counter, status, st); break;
  }
}

}  // namespace symnmf
