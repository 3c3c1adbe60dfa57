// tools/mma_rate.cu -- calibration microbenchmark (not product): issue rate
// of the K12 E-phase UMMA shapes on one SM, operands resident in shared
// memory (no TMA), so the tensor pipe / smem operand path alone is timed.
//   A = [128 x 16] bf16 tile, MN-major (E^T, K12's E phase) or K-major;
//   B = [N x 16] bf16 K-major SWIZZLE_64B (K12's P tiles) or SW128;
//   8 accumulators (sub-tiles), as in the E phase's inner loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_rate.cu -o tools/mma_rate
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2510_08666_b200/csrc/common.cuh"

using namespace dinfer;

__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, int N, int a_mn, int b_sw64, int per_sub,
                                                     unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = smem;              // 64 KB: 16 boxes of [64 x 32] bf16 (K12's E stage layout)
  uint8_t* b = smem + 65536;      // 32 KB: P tile
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536 + 32768);
  uint32_t* misc = reinterpret_cast<uint32_t*>(bar + 2);
  for (int i = threadIdx.x; i < (65536 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3c003c00u, 0, 0x3c003c00u, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    fence_mbar_init();
  }
  fence_proxy_async();
  if (threadIdx.x < 32) tmem_alloc(&misc[0], 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = misc[0];
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16(128, N, a_mn != 0, false);
    const uint32_t ebox = 128u * 32u;
    const uint32_t e_addr = smem_u32(a), phi = smem_u32(b);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
      for (int k = 0; k < 2; ++k) {
        const uint64_t bd = b_sw64 ? sdesc_swz(phi + k * 32, 16, 512, 4) : sdesc_sw128(phi + k * 32, 16, 1024);
        for (int sub = 0; sub < 8; ++sub) {
          const uint64_t ad = a_mn ? sdesc_sw128(e_addr + sub * 2 * ebox + k * 16 * 128, ebox, 1024)
                                   : sdesc_sw128(e_addr + (sub % 4) * 16384 + k * 32, 16, 1024);
          const uint32_t d = tmem + static_cast<uint32_t>(sub * N) % 512u;
          for (int r = 0; r < per_sub; ++r) mma_bf16(d, ad, bd, idesc, (it | k | r) != 0);
        }
      }
    }
    mma_commit(&bar[0]);
    mbar_wait(&bar[0], 0);
    const unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const size_t smem = 65536 + 32768 + 64 + 1024;
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  struct Cfg {
    const char* name;
    int N, a_mn, b_sw64, per_sub;
  } cfgs[] = {
      {"K12 E now: N=32 A MN-major B SW64, hi+lo (2/sub)", 32, 1, 1, 2},
      {"N=32 A MN-major B SW64, 1/sub", 32, 1, 1, 1},
      {"N=64 (hi|lo stacked) A MN-major B SW64, 1/sub", 64, 1, 1, 1},
      {"N=32 A K-major B SW64, 2/sub", 32, 0, 1, 2},
      {"N=64 A K-major B SW64, 1/sub", 64, 0, 1, 1},
      {"N=128 A MN-major, 1/sub", 128, 1, 0, 1},
      {"N=256 A MN-major, 1/sub", 256, 1, 0, 1},
  };
  const int iters = 2000;
  for (auto& c : cfgs) {
    for (int grid : {1, 148}) {
      mma_kernel<<<grid, 128, smem>>>(iters, c.N, c.a_mn, c.b_sw64, c.per_sub, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      const double n_mma = static_cast<double>(iters) * 2 * 8 * c.per_sub;
      const double macs = n_mma * 128.0 * c.N * 16;
      printf("%-52s grid %3d: %6.1f cyc/MMA  %6.0f MAC/cyc/SM  %s\n", c.name, grid, mx / n_mma, macs / mx,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
