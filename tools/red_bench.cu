// Microbenchmark: the rate of global float reductions (SASS RED / REDG) to random 128-byte rows
// inside an L2-sized destination range -- the access pattern of the sampled CSR scatter
// (spmm.cu: sampled_csr_v4).  Each "row op" adds 32 floats (k = 32) into one random 128 B row:
//   v4: 8 lanes x red.global.add.v4.f32, v2: 16 lanes x .v2.f32, v1: 32 lanes x .f32,
//   st: the same rows written with plain 16 B stores (the LSU/L2 cost without the atomic ALU).
//   ld: the same rows gathered with 16 B loads and summed in registers -- the access pattern of the
//       exact CSR product's F gathers (spmm_nnz.cu), 1e8 row gathers like c4's nonzeros.
// Prints row ops/s and lane-instructions per clock per SM (at the SM clock nvidia-smi reports).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/red_bench.cu -o /tmp/red_bench
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ void red4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void red2(float* p, float2 v) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void red1(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// MODE: 4 / 2 / 1 = floats per lane of a red; 0 = plain float4 stores.  ops: row ops in total.
template <int MODE>
__global__ void __launch_bounds__(256) red_kernel(float* __restrict__ Y, uint32_t nrows, int64_t ops, uint32_t seed) {
  constexpr int W = MODE == 0 ? 4 : MODE;     // floats per lane
  constexpr int LPR = 32 / W;                 // lanes per 128 B row
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / LPR;
  const int li = threadIdx.x % LPR;
  for (int64_t o = gtid / LPR; o < ops; o += ngroups) {
    const uint32_t r = mix((uint32_t)o * 2654435761u + seed) % nrows;
    float* p = Y + (int64_t)r * 32 + li * W;
    if constexpr (MODE == 4) red4(p, make_float4(1.f, 1.f, 1.f, 1.f));
    else if constexpr (MODE == 2) red2(p, make_float2(1.f, 1.f));
    else if constexpr (MODE == 1) red1(p, 1.f);
    else *reinterpret_cast<float4*>(p) = make_float4(1.f, 1.f, 1.f, 1.f);
  }
}

// Row gathers: 8 lanes x 16 B per random row, UNR independent rows in flight per lane group.
template <int UNR>
__global__ void __launch_bounds__(256) gather_kernel(const float4* __restrict__ F, uint32_t nrows, int64_t ops,
                                                     uint32_t seed, float4* __restrict__ out) {
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / 8;
  const int li = threadIdx.x % 8;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t o = gtid / 8; o < ops; o += ngroups * UNR) {
    float4 v[UNR];
#pragma unroll
    for (int j = 0; j < UNR; ++j) {
      const int64_t oj = o + j * ngroups;
      const uint32_t r = mix((uint32_t)oj * 2654435761u + seed) % nrows;
      v[j] = oj < ops ? __ldg(F + (int64_t)r * 8 + li) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < UNR; ++j) { acc.x += v[j].x; acc.y += v[j].y; acc.z += v[j].z; acc.w += v[j].w; }
  }
  if (acc.x == 123.456f) out[gtid] = acc;   // keep the loads
}

static void run_gather(const float* Y, uint32_t nrows, int64_t ops, int sms, float* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = sms * 8;
  float best = 1e30f;
  for (int it = 0; it < 4; ++it) {
    cudaEventRecord(e0);
    gather_kernel<8><<<grid, 256>>>(reinterpret_cast<const float4*>(Y), nrows, ops, 5u + it,
                                    reinterpret_cast<float4*>(out));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (it > 0 && ms < best) best = ms;
  }
  printf("ld  rows=%9u (%6.1f MB) ops=%lld  %.3f ms  %.2f G row-gathers/s  %.2f TB/s gathered\n", nrows,
         nrows * 128.0 / 1e6, (long long)ops, best, ops / (best * 1e-3) / 1e9, ops / (best * 1e-3) * 128 / 1e12);
}

template <int MODE>
static void run(const char* name, float* Y, uint32_t nrows, int64_t ops, int sms, double mhz) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = sms * 8;
  red_kernel<MODE><<<grid, 256>>>(Y, nrows, ops, 1u);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int it = 0; it < 5; ++it) {
    cudaEventRecord(e0);
    red_kernel<MODE><<<grid, 256>>>(Y, nrows, ops, 17u + it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const int lanes = MODE == 0 ? 8 : 32 / MODE;
  const double rows_s = ops / (best * 1e-3);
  printf("%-3s rows=%9u (%6.1f MB) ops=%lld  %.3f ms  %.2f G row-ops/s  %.2f TB/s payload  %.3f lane-instr/clk/SM\n",
         name, nrows, nrows * 128.0 / 1e6, (long long)ops, best, rows_s / 1e9, rows_s * 128 / 1e12,
         rows_s * lanes / (sms * mhz * 1e6));
}

int main(int argc, char** argv) {
  const double mhz = argc > 1 ? atof(argv[1]) : 1965.0;
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  const int64_t ops = 12 * 1000 * 1000;   // c4: ~12M sampled nonzeros per half
  const uint32_t sizes[] = {1u << 14, 1u << 17, 675000u, 2000000u};   // 2 MB, 16 MB, 86 MB (one c4 pass), 256 MB
  float* Y; cudaMalloc(&Y, (size_t)2000000 * 128);
  cudaMemset(Y, 0, (size_t)2000000 * 128);
  printf("SMs %d, clock %.0f MHz\n", sms, mhz);
  for (uint32_t nrows : sizes) {
    run<4>("v4", Y, nrows, ops, sms, mhz);
    run<2>("v2", Y, nrows, ops, sms, mhz);
    run<1>("v1", Y, nrows, ops, sms, mhz);
    run<0>("st", Y, nrows, ops, sms, mhz);
  }
  float* out; cudaMalloc(&out, (size_t)sms * 8 * 256 * 16);
  const uint32_t gsizes[] = {1u << 14, 500000u, 1000000u, 2000000u};   // 2 MB, 64 MB, 128 MB, 256 MB (c4's F)
  for (uint32_t nrows : gsizes) run_gather(Y, nrows, 100 * 1000 * 1000, sms, out);
  cudaFree(out);
  cudaFree(Y);
  return cudaGetLastError() != cudaSuccess;
}
