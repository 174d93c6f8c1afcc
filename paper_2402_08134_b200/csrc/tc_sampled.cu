// (a9) The sampled dense product on the 5th-generation tensor cores, in 3xTF32:
//
//   Y_s = A[U, :]^T (Omega F[U, :])      (Alg. LvS-SymNMF P:687-688 / P:694-695, Y_H of the
//                                         sampled NLS problem; A[U,:]^T = A[:,U] by symmetry, Z28)
//
// A n x n fp32 row-major (the sampled rows are contiguous in memory), U = the plan's unique rows
// (|U| <= s), Omega = their weights, F n x k.  The contraction runs over the sampled rows u, so the
// A operand of the MMA -- 128 output rows c x 8 sampled rows u -- is MN-major: a sampled row
// contributes 128 contiguous bytes per 32 output rows.  That is exactly the layout of a row slice
// of A, so the gather needs no transposition: 16-byte cp.async chunks land in MN-major atoms of
// the SWIZZLE_128B_BASE32B layout (4 K-rows x 128 B; the 32-byte chunk j of K-row r at
// (j ^ (r mod 4)) * 32) -- the only MN-major smem layout the tf32 MMA accepts (with the plain
// 128B swizzle the MMA reads zeros; measured).
//
// Per CTA: one 128-row output tile (c0 .. c0+127) and one range of U (split over gridDim.y so the
// grid fills whole waves of the 148 SMs):
//   warps 0..3   producers.  Per stage (32 sampled rows) each thread cp.asyncs its own 8 chunks of
//                the 32 x 512 B slab of A (rows U_u, columns c0..c0+127) and its chunks of the
//                [Omega F]_hi^T / [Omega F]_lo^T tiles (2 NP rows of 128 B, K-major, written once
//                per product by sampled_b_split) into a RAW ring that only this thread touches, SR
//                stages deep.  When its chunks of stage j land it writes A_hi = a & 0xffffe000,
//                A_lo = a - A_hi and the B chunks into one of two MMA slots, fence.proxy.async,
//                arrive.  The raw slot is free again at once, so the loads in flight never wait
//                for the tensor core (a single ring, where the MMA read the raw slot as A_hi, tied
//                every reissue to an MMA round trip: 0.21 ms at c3 against 0.24 ms for SIMT).
//   warp 4       one elected thread issues per K=8 step A_hi [B_hi | B_lo] and A_lo [B_hi | B_lo]
//                (M = 128, N = 2 NP) into independent TMEM accumulators, as tc_gemm.cu does; the
//                accumulators restart every SB_DRAIN k-blocks (the tensor core's truncating fp32
//                accumulate, tc_gemm.cu header)
//   warp 5       TMEM allocation
//   warps 6..9   drain TMEM into fp32 registers; at the end add into Y (fp32 red.add; Y zeroed
//                when U is split, else plain stores)
// A TMA form (one thread issuing 32 tile::gather4 loads per stage through
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) was correct but slower (0.27 ms at c3); not kept.
#include "tc_common.cuh"

#include <cstdlib>
#include <cstring>

namespace symnmf {

namespace {

constexpr int SB_BM = 128;          // output rows per CTA
constexpr int SB_BK = 32;           // sampled rows per stage
constexpr int SB_THREADS = 320;     // 10 warps
constexpr int SB_DRAIN = 16;        // k-blocks per accumulator chunk (tc_gemm.cu)

template <int NP>
struct SbLayout {
  static constexpr uint32_t A_BYTES = SB_BM * SB_BK * 4;              // 16 KB slab
  static constexpr uint32_t B_BYTES = 2 * NP * SB_BK * 4;             // [B_hi ; B_lo] tiles
  static constexpr uint32_t RAW = A_BYTES + B_BYTES;                   // raw ring stage
  static constexpr uint32_t MMA = 2 * A_BYTES + B_BYTES;               // MMA slot: A_hi | A_lo | B
  static constexpr int SR = NP <= 16 ? 6 : NP <= 32 ? 5 : 3;          // raw ring depth
  static constexpr size_t smem = 1024 + (size_t)SR * RAW + 2 * (size_t)MMA + 8 * 8 + 16;
};

}  // namespace

// [Omega F]^T split into tf32 hi / lo parts, K-major: hiT[j * ldu + u] = hi(omega_u F[U_u, j]),
// zero for j >= k and for u in [|U|, ldu).  The product omega_u F is formed in fp64.
__global__ void sampled_b_split(const float* __restrict__ F, int k, int NP, const int32_t* __restrict__ uniq,
                                const double* __restrict__ w, const int64_t* __restrict__ n_uniq_dev, int64_t ldu,
                                float* __restrict__ hiT, float* __restrict__ loT, const int32_t* __restrict__ status) {
  if (dev_failed(status)) return;
  const int64_t nu = *n_uniq_dev;
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= ldu || u >= (nu + SB_BK - 1) / SB_BK * SB_BK) return;
  const bool ok = u < nu;
  const int64_t row = ok ? (int64_t)uniq[u] : 0;
  const double om = ok ? w[u] : 0.0;
  for (int j = 0; j < NP; ++j) {
    const double v = (ok && j < k) ? om * (double)F[row * k + j] : 0.0;
    const float h = __uint_as_float(__float_as_uint((float)v) & 0xFFFFE000u);
    hiT[(int64_t)j * ldu + u] = h;
    loT[(int64_t)j * ldu + u] = (float)(v - (double)h);
  }
}

template <int NP>
__global__ void __launch_bounds__(SB_THREADS, 1)
    tc_sampled_3xtf32(const float* __restrict__ A, int64_t lda, int64_t n, const int32_t* __restrict__ uniq,
                      const int64_t* __restrict__ n_uniq_dev, const float* __restrict__ hiT,
                      const float* __restrict__ loT, int64_t ldu, float* __restrict__ Y, int k,
                      const int32_t* __restrict__ status) {
  using L = SbLayout<NP>;
  constexpr int SR = L::SR;
  constexpr int NACC = NP <= 32 ? 4 : 2;
  constexpr uint32_t ACC_COLS = 2 * NP;
  constexpr uint32_t BUF_COLS = NACC * ACC_COLS;
  constexpr uint32_t TMEM_COLS = 2 * BUF_COLS <= 128 ? 128 : 2 * BUF_COLS <= 256 ? 256 : 512;
  // D fp32, A / B tf32, A MN-major (bit 15), B K-major, N = 2 NP, M = 128
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) |
                             ((uint32_t)((2 * NP) >> 3) << 17) | ((uint32_t)(SB_BM >> 4) << 24);
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  unsigned char* slot = sm;                               // 2 MMA slots
  unsigned char* raw = sm + 2 * L::MMA;                   // SR raw stages
  uint64_t* hl_full = reinterpret_cast<uint64_t*>(raw + SR * L::RAW);   // [2]
  uint64_t* hl_empty = hl_full + 2;                                    // [2]
  uint64_t* acc_full = hl_empty + 2;                                   // [2]
  uint64_t* acc_empty = acc_full + 2;                                  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  if (dev_failed(status)) return;
  const int64_t nu = *n_uniq_dev;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c0 = (int64_t)blockIdx.x * SB_BM;
  // this CTA's k-blocks of 32 sampled rows: an equal share of the |U| / 32 blocks per U split
  const int64_t nkb_all = (nu + SB_BK - 1) / SB_BK;
  const int64_t kb_per_split = (nkb_all + gridDim.y - 1) / gridDim.y;
  const int64_t kb0 = (int64_t)blockIdx.y * kb_per_split;
  const int nkb = (int)min64(kb_per_split, nkb_all - kb0);
  if (nkb <= 0) {   // whole CTA, before any barrier; with |U| = 0 and no split, Y's tile is 0
    if (gridDim.y == 1)
      for (int64_t e = threadIdx.x; e < (int64_t)SB_BM * k; e += blockDim.x)
        if (c0 + e / k < n) Y[c0 * k + e] = 0.f;
    return;
  }

  if (threadIdx.x == 0) {
    for (int h = 0; h < 2; ++h) {
      mbar_init(hl_full + h, 128); mbar_init(hl_empty + h, 1);
      mbar_init(acc_full + h, 1); mbar_init(acc_empty + h, 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    const int t = threadIdx.x;   // 0..127
    // A chunk e = t + 128 q (q < 8): K-row r = e / 32 = t / 32 + 4 q (warp-uniform), 16-B chunk
    // cq = e % 32 = lane of the row's 512 B.  Atom (m block cq / 8, 4-row group r / 4) at
    // (r / 4) * 2048 + (cq / 8) * 512; in it the 32-byte chunk (cq % 8) / 2 of row r % 4 is
    // stored at position ((cq % 8) / 2) ^ (r % 4).
    auto aoff = [](int r, int cq) -> uint32_t {
      const int r4 = r & 3;
      return (uint32_t)((r >> 2) * 2048 + (cq >> 3) * 512 + r4 * 128 + ((((cq & 7) >> 1) ^ r4) << 5) + ((cq & 1) << 4));
    };
    // B chunk e = t + 128 q (q < NP / 8): row nn = e / 8 (< NP: hi, else lo), 16-B chunk e % 8,
    // K-major 128B swizzle
    auto boff = [](int e) -> uint32_t { const int nn = e >> 3, j = e & 7; return (uint32_t)(nn * 128 + ((j ^ (nn & 7)) << 4)); };
    // the sampled row indices of a stage are loaded one stage ahead, off the issue path
    int32_t urow[8];
    auto load_rows = [&](int i) {
      const int64_t ub = (kb0 + i) * SB_BK;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t u = ub + (t >> 5) + 4 * q;
        urow[q] = (i < nkb && u < nu) ? __ldg(uniq + u) : -1;
      }
    };
    auto issue = [&](int i) {
      unsigned char* st = raw + (i % SR) * L::RAW;
      const int64_t ub = (kb0 + i) * SB_BK;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int r = (t >> 5) + 4 * q, cq = t & 31;
        const int64_t c = c0 + 4 * cq;
        const bool ok = urow[q] >= 0 && c < n;
        cp_async16(st + aoff(r, cq), ok ? (const void*)(A + (int64_t)urow[q] * lda + c) : (const void*)A, ok);
      }
#pragma unroll
      for (int q = 0; q < (16 * NP) / 128; ++q) {
        const int e = t + 128 * q, nn = e >> 3, j = e & 7;
        const float* src = (nn < NP ? hiT + (int64_t)nn * ldu : loT + (int64_t)(nn - NP) * ldu) + ub + 4 * j;
        cp_async16(st + L::A_BYTES + boff(e), src, true);
      }
    };
    load_rows(0);
    for (int i = 0; i < nkb + SR - 1; ++i) {
      if (i < nkb) {   // raw slot i % SR: this thread's chunks of stage i - SR were consumed at i - 1
        issue(i);
        load_rows(i + 1);
      }
      cp_async_commit();
      if (i >= SR - 1) {
        const int j = i - (SR - 1), h = j & 1;
        cp_async_wait<SR - 1>();   // this thread's chunks of stage j have landed
        if (j >= 2) mbar_wait(hl_empty + h, ((j >> 1) - 1) & 1);
        const unsigned char* st = raw + (j % SR) * L::RAW;
        unsigned char* ms = slot + h * L::MMA;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t off = aoff((t >> 5) + 4 * q, t & 31);
          const uint4 v = *reinterpret_cast<const uint4*>(st + off);
          uint4 hi, lo;
          hi.x = v.x & 0xFFFFE000u; hi.y = v.y & 0xFFFFE000u; hi.z = v.z & 0xFFFFE000u; hi.w = v.w & 0xFFFFE000u;
          lo.x = __float_as_uint(__uint_as_float(v.x) - __uint_as_float(hi.x));
          lo.y = __float_as_uint(__uint_as_float(v.y) - __uint_as_float(hi.y));
          lo.z = __float_as_uint(__uint_as_float(v.z) - __uint_as_float(hi.z));
          lo.w = __float_as_uint(__uint_as_float(v.w) - __uint_as_float(hi.w));
          *reinterpret_cast<uint4*>(ms + off) = hi;
          *reinterpret_cast<uint4*>(ms + L::A_BYTES + off) = lo;
        }
#pragma unroll
        for (int q = 0; q < (16 * NP) / 128; ++q) {
          const uint32_t off = boff(t + 128 * q);
          *reinterpret_cast<uint4*>(ms + 2 * L::A_BYTES + off) = *reinterpret_cast<const uint4*>(st + L::A_BYTES + off);
        }
        fence_proxy_async();
        mbar_arrive(hl_full + h);
      }
    }
    cp_async_wait<0>();
  } else if (warp == 4) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int h = i & 1;
        const int c = i / SB_DRAIN, b = c & 1;
        if (i % SB_DRAIN == 0 && c >= 2) mbar_wait(acc_empty + b, ((c >> 1) - 1) & 1);
        mbar_wait(hl_full + h, (i >> 1) & 1);
        tc_fence_after();
        const uint32_t a_hi = smem_u32(slot + h * L::MMA), a_lo = a_hi + L::A_BYTES, bb = a_hi + 2 * L::A_BYTES;
        const uint32_t td = tmem + (uint32_t)b * BUF_COLS;
#pragma unroll
        for (int kk = 0; kk < SB_BK / 8; ++kk) {
          const uint32_t acc0 = ((i % SB_DRAIN) != 0 || kk >= (NACC == 4 ? 2 : 1)) ? 1u : 0u;
          const uint32_t tq = td + (NACC == 4 ? (uint32_t)(kk & 1) * 2 * ACC_COLS : 0u);
          // K step kk = rows 8kk .. 8kk+7 = 4-row groups 2kk, 2kk+1 (SBO apart), 4 M atoms (LBO apart)
          mma_tf32(tq, smem_desc_mn128_b32(a_hi + kk * 4096, 512, 2048), smem_desc_k128(bb + kk * 32), IDESC, acc0);
          mma_tf32(tq + ACC_COLS, smem_desc_mn128_b32(a_lo + kk * 4096, 512, 2048), smem_desc_k128(bb + kk * 32),
                   IDESC, acc0);
        }
        mma_commit(hl_empty + h);
        if ((i + 1) % SB_DRAIN == 0 || i + 1 == nkb) mma_commit(acc_full + b);
      }
    }
  } else if (warp >= 6) {
    const int wq = warp & 3;   // TMEM lane quarter this warp may access
    float acc[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) acc[j] = 0.f;
    const int nch = (nkb + SB_DRAIN - 1) / SB_DRAIN;
    for (int c = 0; c < nch; ++c) {
      const int b = c & 1;
      mbar_wait_sleep(acc_full + b, (c >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < NACC * 2 * NP; cc += 16) {
        const int cb = cc % NP;
        uint32_t r[16];
        const uint32_t taddr = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)b * BUF_COLS + (uint32_t)cc;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[cb + j] += __uint_as_float(r[j]);
      }
      tc_fence_before();
      mbar_arrive(acc_empty + b);
    }
    const int64_t row = c0 + wq * 32 + lane;
    if (row < n) {
      if (gridDim.y > 1) {
#pragma unroll
        for (int j = 0; j < NP; ++j)
          if (j < k) atomicAdd(Y + row * k + j, acc[j]);
      } else {
#pragma unroll
        for (int j = 0; j < NP; ++j)
          if (j < k) Y[row * k + j] = acc[j];
      }
    }
  }
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

// ---------------------------------------------------------------- host side
static int sb_np(int k) { return k <= 16 ? 16 : k <= 32 ? 32 : 64; }
static int64_t sb_ldu(int64_t cap) { return (cap + SB_BK - 1) / SB_BK * SB_BK; }

// SYMNMF_SAMPLED_DENSE=simt selects the fp32 SIMT kernel (dense.cu), =tc this one wherever it applies;
// by default this one from n = 16384 (c1, n = 1,000: the SIMT kernel's single launch is faster than the
// split + zero + tensor-core launches, 10.4k vs 11.9k LvS it/s) (symnmf.h).
bool sampled_dense_tc_enabled(int64_t n) {
  const char* e = getenv("SYMNMF_SAMPLED_DENSE");
  if (e && !strcmp(e, "simt")) return false;
  if (e && !strcmp(e, "tc")) return true;
  return n >= 16384;
}

size_t sampled_dense_tc_scratch(int64_t cap, int k) {
  return k > 64 ? 0 : sizeof(float) * 2 * (size_t)sb_np(k) * sb_ldu(cap) + 256;
}

bool sampled_dense_tc_supported(const float* A, int64_t lda, int64_t n, int k) {
  return k <= 64 && lda % 4 == 0 && n % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
}

template <int NP>
static void launch_sb_t(const float* A, int64_t lda, int64_t n, const float* F, int k, const int32_t* uniq,
                        const double* w, const int64_t* nu, int64_t cap, int64_t u_hint, float* Y, void* scratch,
                        const int32_t* status, cudaStream_t st) {
  using L = SbLayout<NP>;
  const int64_t ldu = sb_ldu(cap);
  float* hiT = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(scratch) + 255) & ~uintptr_t(255));
  float* loT = hiT + (size_t)NP * ldu;
  sampled_b_split<<<(unsigned)((ldu + 255) / 256), 256, 0, st>>>(F, k, NP, uniq, w, nu, ldu, hiT, loT, status);
  // U splits: whole waves of one CTA per SM over (output tiles x U ranges), for the expected |U|
  // (u_hint), at least 4 k-blocks per CTA; the kernel divides the actual |U| (on the device)
  const int64_t mt = (n + SB_BM - 1) / SB_BM;
  const int64_t nkb = (std::min(u_hint, ldu) + SB_BK - 1) / SB_BK;
  int64_t splits = 1;
  double best = 0.0;
  const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(32, nkb / 4));
  for (int64_t sp = 1; sp <= smax; ++sp) {
    const int64_t ctas = mt * sp, waves = (ctas + 147) / 148;
    const double eff = (double)ctas / (double)(waves * 148) * (1.0 - 0.01 * (double)sp);
    if (eff > best + 1e-9) { best = eff; splits = sp; }
  }
  if (const char* e = getenv("SYMNMF_SB_SPLITS")) splits = std::max(1, atoi(e));   // measurement knob
  if (splits > 1) cudaMemsetAsync(Y, 0, sizeof(float) * n * k, st);
  cudaFuncSetAttribute(tc_sampled_3xtf32<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::smem);
  tc_sampled_3xtf32<NP><<<dim3((unsigned)mt, (unsigned)splits), SB_THREADS, L::smem, st>>>(
      A, lda, n, uniq, nu, hiT, loT, ldu, Y, k, status);
}

void launch_sampled_dense_tc(const float* A, int64_t lda, int64_t n, const float* F, int k, const int32_t* uniq,
                             const double* w, const int64_t* n_uniq_dev, int64_t cap, int64_t u_hint, float* Y,
                             void* scratch, const int32_t* status, cudaStream_t st) {
  switch (sb_np(k)) {
    case 16: launch_sb_t<16>(A, lda, n, F, k, uniq, w, n_uniq_dev, cap, u_hint, Y, scratch, status, st); break;
    case 32: launch_sb_t<32>(A, lda, n, F, k, uniq, w, n_uniq_dev, cap, u_hint, Y, scratch, status, st); break;
    default: launch_sb_t<64>(A, lda, n, F, k, uniq, w, n_uniq_dev, cap, u_hint, Y, scratch, status, st); break;
  }
}

}  // namespace symnmf
