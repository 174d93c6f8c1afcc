// (a10)/(a12) Dense Y = A X on the 5th-generation tensor cores in 3xTF32
// (precision SYMNMF_3XTF32): A n x n fp32 (the data matrix, streamed once from
// HBM), X n x k fp32 (the factor F, or Omega / Q in the range finder).
//
//   Y = A_hi X_hi + A_hi X_lo + A_lo X_hi (+ A_lo X_lo, free),   v_hi = v with the low 13
//   mantissa bits cleared (exactly representable in tf32), v_lo = v - v_hi (exact).
//
// Per CTA (one 128-row tile of A and one K range, split-K over gridDim.y):
//   warp 0      TMA producer: A tile [128 x 32] fp32 (128B swizzle), X_hi^T / X_lo^T tiles
//               [NP x 32] (pre-split and transposed once per product, K-major)
//   warps 4..7  form A_lo = a - (a & 0xffffe000) of the A tile in a second buffer (the raw tile
//               is A_hi: the tf32 MMA ignores the low 13 mantissa bits),
//               fence.proxy.async, arrive
//   warps 8..11 every TC_DRAIN k-blocks drain the TMEM accumulator into fp32 registers
//               (tcgen05.ld, round-to-nearest adds); at the end add the registers into Y
//               (fp32 red.add).  Warp w reads TMEM lanes 32 (w % 4) .. +31.
//   warp 1      one elected thread issues 2 x 4 tcgen05.mma.kind::tf32 (M=128, N=2 NP, K=8)
//               per stage, A_hi [X_hi | X_lo] and A_lo [X_hi | X_lo] with B = the X_hi and X_lo
//               tiles stacked (adjacent in the stage), into two independent accumulators
//               (NP <= 64; one for NP > 64).  Three dependent N = NP MMAs per K=8 step were
//               measured to bound the kernel (1.006 ms at c3 vs 0.647 ms with one MMA): small-N
//               MMAs into one accumulator serialise on the MMA latency.  Chunk c of TC_DRAIN
//               k-blocks uses buffer c & 1, restarting from zero; the stage is committed back to
//               the producer
//   warp 2      TMEM allocation / deallocation
// Pipeline: 3-5 smem stages with full (TMA tx) / conv (128 arrivals) / empty (MMA commit)
// mbarriers, two accumulator buffers with acc_full (MMA commit) / acc_empty (128 arrivals).
//
// Why the drain: the tensor core's fp32 accumulation does not round to nearest -- each MMA's
// add into the accumulator loses about one accumulator ulp, always towards zero.  Measured on
// B200 with one accumulator per K range: a relative bias of -7e-7 per 32-wide k-block of chain,
// -2.1e-4 at n = 30,000 (313 k-blocks per split).  Restarting the accumulator every TC_DRAIN
// k-blocks bounds the bias by the chain length of one chunk; the chunks are summed in registers.
// Measured (tools/tc_bias.py, uniform [0,1) A and X, n = 30,000): mean relative error -1.6e-6,
// max 2.1e-6 with TC_DRAIN = 16 (fp32 SGEMM: max 1.4e-5); TC_DRAIN = 8 / 32: -8e-7 / -3.2e-6 at
// 0.902 / 0.876 ms against 0.886 ms.
#include <cudaTypedefs.h>
#include "tc_common.cuh"

namespace symnmf {

constexpr int TC_BM = 128;
constexpr int TC_BK = 32;          // fp32 elements per 128-byte row
template <int NP> constexpr int tc_stages() { return NP <= 32 ? 5 : NP <= 80 ? 4 : 3; }
constexpr int TC_THREADS = 384;
constexpr int TC_DRAIN = 16;       // k-blocks per accumulator chunk

template <int NP>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_gemm_3xtf32(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapBhi,
                   const __grid_constant__ CUtensorMap mapBlo, int64_t n, int kb_per_split, int64_t nkb_total,
                   float* __restrict__ Y, int64_t ldy, int k, const int32_t* __restrict__ status) {
  constexpr uint32_t A_BYTES = TC_BM * TC_BK * 4;   // 16 KB
  constexpr uint32_t B_BYTES = NP * TC_BK * 4;      // NP x 128 B
  constexpr uint32_t STAGE = 2 * A_BYTES + 2 * B_BYTES;
  // accumulators: NACC independent chains per buffer, each 2 NP columns ([.. X_hi | .. X_lo]);
  // two buffers.  NACC = 4: {A_hi, A_lo} x {even, odd K=8 step}; 2: {A_hi, A_lo}; 1: shared.
  constexpr int NACC = NP <= 32 ? 4 : NP <= 64 ? 2 : 1;
  // NP > 64 (the c5 range finder, NP = 80): A_hi [X_hi | X_lo] (N = 2 NP) and A_lo X_hi (N = NP) into
  // two independent accumulators per buffer (3 NP columns) instead of one chain of two N = 2 NP MMAs,
  // whose A_lo X_lo quarter of the tensor work is dropped (it is below the 3xTF32 error anyway)
  constexpr bool SPLIT2 = NP > 64 && 6 * NP <= 512;
  constexpr uint32_t ACC_COLS = 2 * NP;
  constexpr uint32_t BUF_COLS = SPLIT2 ? 3 * NP : NACC * ACC_COLS;
  constexpr uint32_t IDESC_LO = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NP >> 3) << 17) |
                                ((uint32_t)(TC_BM >> 4) << 24);
  constexpr uint32_t TMEM_COLS = 2 * BUF_COLS <= 128 ? 128 : 2 * BUF_COLS <= 256 ? 256 : 512;
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)((2 * NP) >> 3) << 17) |
                             ((uint32_t)(TC_BM >> 4) << 24);
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + tc_stages<NP>() * STAGE);
  uint64_t* conv = full + tc_stages<NP>();
  uint64_t* empty = conv + tc_stages<NP>();
  uint64_t* acc_full = empty + tc_stages<NP>();   // [2]
  uint64_t* acc_empty = acc_full + 2;             // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  if (dev_failed(status)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.x * TC_BM;
  const int64_t kb0 = (int64_t)blockIdx.y * kb_per_split;
  const int nkb = (int)min64(kb_per_split, nkb_total - kb0);
  if (nkb <= 0) return;

  if (threadIdx.x == 0) {
    for (int s = 0; s < tc_stages<NP>(); ++s) { mbar_init(full + s, 1); mbar_init(conv + s, 128); mbar_init(empty + s, 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(acc_full + b, 1); mbar_init(acc_empty + b, 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % tc_stages<NP>();
        if (i >= tc_stages<NP>()) mbar_wait(empty + s, ((i / tc_stages<NP>()) - 1) & 1);
        unsigned char* st = sm + s * STAGE;
        const int kx = (int)((kb0 + i) * TC_BK);
        mbar_expect_tx(full + s, A_BYTES + 2 * B_BYTES);
        tma_load_2d(&mapA, full + s, st, kx, (int)m0);
        tma_load_2d(&mapBhi, full + s, st + 2 * A_BYTES, kx, 0);
        tma_load_2d(&mapBlo, full + s, st + 2 * A_BYTES + B_BYTES, kx, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % tc_stages<NP>();
        const int c = i / TC_DRAIN, b = c & 1;
        if (i % TC_DRAIN == 0 && c >= 2) mbar_wait(acc_empty + b, ((c >> 1) - 1) & 1);
        mbar_wait(conv + s, (i / tc_stages<NP>()) & 1);
        tc_fence_after();
        const uint32_t a_hi = smem_u32(sm + s * STAGE), a_lo = a_hi + A_BYTES;
        const uint32_t b_hi = a_hi + 2 * A_BYTES, b_lo = b_hi + B_BYTES;
        const uint32_t td = tmem + (uint32_t)b * BUF_COLS;
        if constexpr (SPLIT2) {
#pragma unroll
          for (int kk = 0; kk < TC_BK / 8; ++kk) {
            const uint32_t off = kk * 32;
            const uint32_t acc0 = ((i % TC_DRAIN) != 0 || kk > 0) ? 1u : 0u;
            mma_tf32(td, smem_desc_k128(a_hi + off), smem_desc_k128(b_hi + off), IDESC, acc0);
            mma_tf32(td + 2 * NP, smem_desc_k128(a_lo + off), smem_desc_k128(b_hi + off), IDESC_LO, acc0);
          }
        } else
#pragma unroll
        for (int kk = 0; kk < TC_BK / 8; ++kk) {
          const uint32_t off = kk * 32;   // 8 tf32 = 32 bytes along the swizzled row
          const uint32_t acc0 = ((i % TC_DRAIN) != 0 || kk >= (NACC == 4 ? 2 : 1)) ? 1u : 0u;
          // B = [X_hi; X_lo] (2 NP rows, contiguous in the stage): A_hi [X_hi | X_lo] and
          // A_lo [X_hi | X_lo], into independent accumulators when they fit (NP <= 64)
          const uint32_t tq = td + (NACC == 4 ? (uint32_t)(kk & 1) * 2 * ACC_COLS : 0u);
          mma_tf32(tq, smem_desc_k128(a_hi + off), smem_desc_k128(b_hi + off), IDESC, acc0);
          mma_tf32(tq + (NACC >= 2 ? ACC_COLS : 0u), smem_desc_k128(a_lo + off), smem_desc_k128(b_hi + off), IDESC,
                   NACC >= 2 ? acc0 : 1u);
        }
        mma_commit(empty + s);
        if ((i + 1) % TC_DRAIN == 0 || i + 1 == nkb) mma_commit(acc_full + b);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    const int t = threadIdx.x - 128;   // 0..127
    for (int i = 0; i < nkb; ++i) {
      const int s = i % tc_stages<NP>();
      mbar_wait(full + s, (i / tc_stages<NP>()) & 1);
      uint4* a = reinterpret_cast<uint4*>(sm + s * STAGE);
      uint4* lo = reinterpret_cast<uint4*>(sm + s * STAGE + A_BYTES);
      // A_hi is the raw tile: kind::tf32 reads an fp32 operand's top 19 bits (the low 13
      // mantissa bits are ignored), i.e. exactly a & 0xffffe000; only A_lo is written.
#pragma unroll 4
      for (int e = t; e < (int)(A_BYTES / 16); e += 128) {
        const uint4 v = a[e];
        uint4 l;
        l.x = __float_as_uint(__uint_as_float(v.x) - __uint_as_float(v.x & 0xFFFFE000u));
        l.y = __float_as_uint(__uint_as_float(v.y) - __uint_as_float(v.y & 0xFFFFE000u));
        l.z = __float_as_uint(__uint_as_float(v.z) - __uint_as_float(v.z & 0xFFFFE000u));
        l.w = __float_as_uint(__uint_as_float(v.w) - __uint_as_float(v.w & 0xFFFFE000u));
        lo[e] = l;
      }
      fence_proxy_async();
      mbar_arrive(conv + s);
    }
  } else if (warp >= 8) {
    const int wq = warp & 3;
    float acc[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) acc[j] = 0.f;
    // drain chunk c: TMEM lane = tile row, column = output column
    auto drain = [&](int c) {
      const int b = c & 1;
      mbar_wait_sleep(acc_full + b, (c >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < (int)BUF_COLS; cc += 16) {
        const int c0 = cc % NP;   // column block of Y; the NACC x {X_hi, X_lo} partial sums add up
        uint32_t r[16];
        const uint32_t taddr = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)b * BUF_COLS + (uint32_t)cc;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[c0 + j] += __uint_as_float(r[j]);
      }
      tc_fence_before();
      mbar_arrive(acc_empty + b);
    };
    const int nch = (nkb + TC_DRAIN - 1) / TC_DRAIN;
    for (int c = 0; c < nch; ++c) drain(c);
    const int64_t row = m0 + wq * 32 + lane;
    if (row < n) {
#pragma unroll
      for (int j = 0; j < NP; ++j)
        if (j < k) atomicAdd(Y + row * ldy + j, acc[j]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

// X (n x k, ldx) -> X_hi^T, X_lo^T (NP x ldk, K contiguous, zero padded)
__global__ void split_transpose(const float* __restrict__ X, int64_t ldx, int64_t n, int k, int NP, int64_t ldk,
                                float* __restrict__ hiT, float* __restrict__ loT) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ldk) return;
  for (int c = 0; c < NP; ++c) {
    float v = (j < n && c < k) ? X[j * ldx + c] : 0.f;
    const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    hiT[(int64_t)c * ldk + j] = h;
    loT[(int64_t)c * ldk + j] = v - h;
  }
}

// ---------------------------------------------------------------- host side
static int np_for(int k) { return k <= 16 ? 16 : k <= 32 ? 32 : k <= 64 ? 64 : k <= 80 ? 80 : 96; }
static int64_t ldk_for(int64_t n) { return (n + 31) / 32 * 32; }

size_t dense_ah_tc_scratch(int64_t n, int k) { return sizeof(float) * 2 * (size_t)np_for(k) * ldk_for(n) + 1024; }

template <int NP>
static bool launch_tc_t(const float* A, int64_t lda, int64_t n, const float* X, int64_t ldx, int k, float* Y,
                        int64_t ldy, void* scratch, const int32_t* status, cudaStream_t st) {
  const int64_t ldk = ldk_for(n);
  float* hiT = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(scratch) + 255) & ~uintptr_t(255));
  float* loT = hiT + (size_t)NP * ldk;
  CUtensorMap mA, mH, mL;
  if (!make_map(&mA, A, (uint64_t)n, (uint64_t)n, (uint64_t)lda * 4, TC_BK, TC_BM)) return false;
  if (!make_map(&mH, hiT, (uint64_t)ldk, (uint64_t)NP, (uint64_t)ldk * 4, TC_BK, NP)) return false;
  if (!make_map(&mL, loT, (uint64_t)ldk, (uint64_t)NP, (uint64_t)ldk * 4, TC_BK, NP)) return false;
  split_transpose<<<(unsigned)((ldk + 255) / 256), 256, 0, st>>>(X, ldx, n, k, NP, ldk, hiT, loT);
  cudaMemset2DAsync(Y, sizeof(float) * ldy, 0, sizeof(float) * k, n, st);
  const int64_t mt = (n + TC_BM - 1) / TC_BM;
  const int64_t nkb = (n + TC_BK - 1) / TC_BK;
  int64_t splits = std::max<int64_t>(1, (148 * 4 + mt - 1) / mt);
  splits = std::min<int64_t>(splits, nkb);
  const int kps = (int)((nkb + splits - 1) / splits);
  splits = (nkb + kps - 1) / kps;
  constexpr size_t STAGE = 2 * TC_BM * TC_BK * 4 + 2 * NP * TC_BK * 4;
  const size_t smem = 1024 + tc_stages<NP>() * STAGE + (3 * tc_stages<NP>() + 4) * 8 + 16;
  cudaFuncSetAttribute(tc_gemm_3xtf32<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tc_gemm_3xtf32<NP><<<dim3((unsigned)mt, (unsigned)splits), TC_THREADS, smem, st>>>(mA, mH, mL, n, kps, nkb, Y, ldy,
                                                                                     k, status);
  return true;
}

bool launch_dense_ah_tc(const float* A, int64_t lda, int64_t n, const float* X, int64_t ldx, int k, float* Y,
                        int64_t ldy, void* scratch, size_t scratch_bytes, const int32_t* status, cudaStream_t st) {
  if (lda % 4 != 0 || (reinterpret_cast<uintptr_t>(A) & 15) || k > 96) return false;
  if (!scratch || scratch_bytes < dense_ah_tc_scratch(n, k)) return false;
  switch (np_for(k)) {
    case 16: return launch_tc_t<16>(A, lda, n, X, ldx, k, Y, ldy, scratch, status, st);
    case 32: return launch_tc_t<32>(A, lda, n, X, ldx, k, Y, ldy, scratch, status, st);
    case 64: return launch_tc_t<64>(A, lda, n, X, ldx, k, Y, ldy, scratch, status, st);
    case 80: return launch_tc_t<80>(A, lda, n, X, ldx, k, Y, ldy, scratch, status, st);
    default: return launch_tc_t<96>(A, lda, n, X, ldx, k, Y, ldy, scratch, status, st);
  }
}

}  // namespace symnmf
