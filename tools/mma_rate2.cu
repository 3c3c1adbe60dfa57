// tools/mma_rate2.cu -- tcgen05.mma issue cost (not product): the same UMMA
// (M = 128, N = 32 / 64 / 256, A MN-major, B SW64/SW128) issued
//   (a) by one thread of a divergent branch (K12's style: the compiler wraps
//       every UTCHMMA in an ELECT / R2UR.BROADCAST waterfall), or
//   (b) by the whole warp with elect.sync inside the asm (operands uniform).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_rate2.cu -o tools/mma_rate2
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2510_08666_b200/csrc/common.cuh"

using namespace dinfer;

__device__ __forceinline__ void mma_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

template <int MODE>  // 0: single thread, 8 accumulators; 1: warp-issued, 8 accumulators
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, int N, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 98304);
  uint32_t* misc = reinterpret_cast<uint32_t*>(bar + 2);
  for (int i = threadIdx.x; i < 98304 / 16; i += blockDim.x)
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
  const uint32_t idesc = idesc_bf16(128, N, true, false);
  const uint32_t ebox = 128u * 32u;
  const uint32_t e_addr = smem_u32(smem), phi = smem_u32(smem + 65536);
  if (MODE == 0) {
    if (threadIdx.x == 0) {
      const unsigned long long t0 = clock64();
      for (int it = 0; it < iters; ++it)
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int sub = 0; sub < 8; ++sub)
            mma_bf16(tmem + static_cast<uint32_t>(sub * N) % 512u,
                     sdesc_sw128(e_addr + sub * 2 * ebox + k * 16 * 128, ebox, 1024),
                     sdesc_swz(phi + k * 32, 16, 512, 4), idesc, (it | k) != 0);
      mma_commit(&bar[0]);
      mbar_wait(&bar[0], 0);
      out[blockIdx.x] = clock64() - t0;
    }
  } else {
    if (threadIdx.x < 32) {
      const unsigned long long t0 = clock64();
      for (int it = 0; it < iters; ++it)
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int sub = 0; sub < 8; ++sub)
            mma_warp(tmem + static_cast<uint32_t>(sub * N) % 512u,
                     sdesc_sw128(e_addr + sub * 2 * ebox + k * 16 * 128, ebox, 1024),
                     sdesc_swz(phi + k * 32, 16, 512, 4), idesc, (it | k) != 0);
      commit_warp(&bar[0]);
      mbar_wait(&bar[0], 0);
      if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const size_t smem = 98304 + 64 + 1024;
  cudaFuncSetAttribute(mma_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaFuncSetAttribute(mma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  const int iters = 2000;
  for (int mode = 0; mode < 2; ++mode)
    for (int N : {32, 64, 128, 256})
      for (int grid : {1, 148}) {
        if (mode == 0) mma_kernel<0><<<grid, 128, smem>>>(iters, N, d);
        else mma_kernel<1><<<grid, 128, smem>>>(iters, N, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        const double n_mma = static_cast<double>(iters) * 16;
        printf("%s N=%3d grid %3d: %6.1f cyc/MMA  %6.0f MAC/cyc/SM %s\n", mode ? "warp-issued " : "one thread  ", N,
               grid, mx / n_mma, n_mma * 128.0 * N * 16 / mx, e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
