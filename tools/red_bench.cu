// tools/red_bench.cu -- calibration microbenchmark (not part of the product):
// cost of the L2 bulk reductions (cp.reduce.async.bulk .add) that merge the
// per-CTA smoothing partials of K12 into one [M x H] record.  148 CTAs each
// reduce a [32 x 1024] slice (half the hidden columns, like K12's hidden-slice
// CTAs) into a shared [32 x 2048] accumulator: fp32 .add.f32 (128 KB per CTA)
// and fixed-point .add.u64 (256 KB per CTA, deterministic), all CTAs at once
// (worst case) and staggered.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/red_bench.cu -o tools/red_bench
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "../paper_2510_08666_b200/csrc/common.cuh"

using namespace dinfer;

template <typename T>
__device__ __forceinline__ void bulk_red(void* gdst, const void* ssrc, uint32_t bytes) {
  if constexpr (sizeof(T) == 4)
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
  else
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
}

// rows x cols elements of T per CTA, staged in `chunk_cols` column pieces
template <typename T>
__global__ void red_kernel(T* acc, int H, int rows, int cols, int chunk_cols, unsigned delay_ns,
                           unsigned long long* t_out) {
  extern __shared__ uint8_t smem_raw[];
  T* tile = reinterpret_cast<T*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const int hs = blockIdx.x & 1;
  if (delay_ns) {
    const unsigned long long t0 = globaltimer_ns();
    while (globaltimer_ns() - t0 < static_cast<unsigned long long>(delay_ns) * (blockIdx.x % 16)) {
    }
  }
  const unsigned long long ts = globaltimer_ns();
  for (int c0 = 0; c0 < cols; c0 += chunk_cols) {
    for (int i = threadIdx.x; i < rows * chunk_cols; i += blockDim.x) tile[i] = static_cast<T>(1);
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x < rows)
      bulk_red<T>(acc + static_cast<long>(threadIdx.x) * H + hs * cols + c0, tile + threadIdx.x * chunk_cols,
                  chunk_cols * sizeof(T));
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    t_out[2 * blockIdx.x] = ts;
    t_out[2 * blockIdx.x + 1] = globaltimer_ns();
  }
}

// thread-issued reductions straight from registers: lane = hidden column,
// like a TMEM load (tcgen05.ld 32x32b: thread = lane = h, 32 columns = s);
// V4: staged through smem and issued as red.global.add.v4.f32
template <bool V4>
__global__ void red_thr_kernel(float* acc, int H, int rows, int cols, unsigned delay_ns, unsigned long long* t_out) {
  __shared__ float tile[32][129];
  const int hs = blockIdx.x & 1;
  if (delay_ns) {
    const unsigned long long t0 = globaltimer_ns();
    while (globaltimer_ns() - t0 < static_cast<unsigned long long>(delay_ns) * (blockIdx.x % 16)) {
    }
  }
  const unsigned long long ts = globaltimer_ns();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // 8 warps: warp w covers columns [w*128, w*128+128) of the CTA's 1024
  for (int c = warp * 128; c < cols; c += 8 * 128) {
    float x[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = 1.f + 1e-3f * lane;
    if (!V4) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int j = 0; j < 32; ++j)
          atomicAdd(acc + static_cast<long>(j) * H + hs * cols + c + q * 32 + lane, x[j]);
    } else {
      for (int q = 0; q < 4; ++q) {
        float* gcol = acc + hs * cols + c + q * 32;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {  // rows j..j+3: lane l writes row j + l/8, columns 4*(l%8)..
          const int r = j + (lane >> 3), cc = (lane & 7) * 4;
          const float4 v = make_float4(x[j], x[j], x[j], x[j]);
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(gcol + static_cast<long>(r) * H + cc),
                       "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                       : "memory");
          (void)tile;
        }
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    t_out[2 * blockIdx.x] = ts;
    t_out[2 * blockIdx.x + 1] = globaltimer_ns();
  }
}

template <bool V4>
void run_thr(const char* name, unsigned delay) {
  const int H = 2048, rows = 32, cols = 1024, grid = 148;
  float* acc;
  cudaMalloc(&acc, static_cast<size_t>(rows) * H * 4);
  unsigned long long* t;
  cudaMalloc(&t, grid * 16);
  std::vector<unsigned long long> th(2 * grid);
  double span_us = 0, cta_us = 0;
  std::vector<float> ms;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int r = 0; r < 13; ++r) {
    cudaMemset(acc, 0, static_cast<size_t>(rows) * H * 4);
    cudaEventRecord(e0);
    red_thr_kernel<V4><<<grid, 256>>>(acc, H, rows, cols, delay, t);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float x;
    cudaEventElapsedTime(&x, e0, e1);
    if (r) {
      ms.push_back(x);
      cudaMemcpy(th.data(), t, grid * 16, cudaMemcpyDeviceToHost);
      unsigned long long lo = ~0ull, hi = 0;
      double sum = 0;
      for (int b = 0; b < grid; ++b) {
        lo = std::min(lo, th[2 * b]);
        hi = std::max(hi, th[2 * b + 1]);
        sum += (th[2 * b + 1] - th[2 * b]) / 1e3;
      }
      span_us += (hi - lo) / 1e3;
      cta_us += sum / grid;
    }
  }
  std::sort(ms.begin(), ms.end());
  const double bytes = static_cast<double>(grid) * rows * cols * 4;
  printf("%-34s            : kernel %7.1f us  reduce span %6.1f us  per-CTA %6.1f us  (%.0f GB/s)  %s\n", name,
         ms[ms.size() / 2] * 1e3, span_us / 12, cta_us / 12, bytes / (span_us / 12 * 1e-6) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(acc);
  cudaFree(t);
}

template <typename T>
void run(const char* name, int chunk_cols, unsigned delay) {
  const int H = 2048, rows = 32, cols = 1024, grid = 148;
  T* acc;
  cudaMalloc(&acc, static_cast<size_t>(rows) * H * sizeof(T));
  unsigned long long* t;
  cudaMalloc(&t, grid * 16);
  const size_t smem = static_cast<size_t>(rows) * chunk_cols * sizeof(T) + 128;
  cudaFuncSetAttribute(red_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> ms;
  std::vector<unsigned long long> th(2 * grid);
  double span_us = 0, cta_us = 0;
  for (int r = 0; r < 13; ++r) {
    cudaMemset(acc, 0, static_cast<size_t>(rows) * H * sizeof(T));
    cudaEventRecord(e0);
    red_kernel<T><<<grid, 256, smem>>>(acc, H, rows, cols, chunk_cols, delay, t);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float x;
    cudaEventElapsedTime(&x, e0, e1);
    if (r) {
      ms.push_back(x);
      cudaMemcpy(th.data(), t, grid * 16, cudaMemcpyDeviceToHost);
      unsigned long long lo = ~0ull, hi = 0;
      double sum = 0;
      for (int b = 0; b < grid; ++b) {
        lo = std::min(lo, th[2 * b]);
        hi = std::max(hi, th[2 * b + 1]);
        sum += (th[2 * b + 1] - th[2 * b]) / 1e3;
      }
      span_us += (hi - lo) / 1e3;
      cta_us += sum / grid;
    }
  }
  std::sort(ms.begin(), ms.end());
  T h[4];
  cudaMemcpy(h, acc, sizeof(h), cudaMemcpyDeviceToHost);
  const double bytes = static_cast<double>(grid) * rows * cols * sizeof(T);
  printf("%-34s chunk %4d cols: kernel %7.1f us  reduce span %6.1f us  per-CTA %6.1f us  (%.0f GB/s)  acc[0]=%g\n",
         name, chunk_cols, ms[ms.size() / 2] * 1e3, span_us / 12, cta_us / 12, bytes / (span_us / 12 * 1e-6) / 1e9,
         static_cast<double>(h[0]));
  cudaFree(acc);
  cudaFree(t);
}

int main() {
  run<float>("f32 all at once", 1024, 0);
  run<float>("f32 all at once", 512, 0);
  run<float>("f32 staggered 1us x (b%16)", 1024, 1000);
  run<unsigned long long>("u64 all at once", 512, 0);
  run<unsigned long long>("u64 all at once", 256, 0);
  run<unsigned long long>("u64 staggered 1us x (b%16)", 512, 1000);
  run_thr<false>("thread red.f32 all at once", 0);
  run_thr<false>("thread red.f32 staggered", 1000);
  run_thr<true>("thread red.v4.f32 all at once", 0);
  run_thr<true>("thread red.v4.f32 staggered", 1000);
  return 0;
}
