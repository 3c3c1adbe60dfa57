// tools/hbm_stream.cu -- calibration microbenchmark (not part of the product):
// how fast can one CTA per SM stream a bf16 matrix through a TMA ring with no
// compute?  Sweeps ring depth and stage size; reports GB/s of pure reads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/hbm_stream.cu -o tools/hbm_stream
//   ./tools/hbm_stream [rows=157184] [cols=2048]
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2510_08666_b200/csrc/common.cuh"

using namespace dinfer;

__global__ void __launch_bounds__(64, 1)
    stream_kernel(const __grid_constant__ CUtensorMap map, int rows, int cols, int stages, int boxes_per_stage,
                  unsigned long long* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t box_bytes = 128u * 128u;  // [128 rows x 64 cols] bf16
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * boxes_per_stage * box_bytes);
  const int r0 = static_cast<int>(static_cast<long>(blockIdx.x) * (rows / 128) / gridDim.x) * 128;
  const int r1 = static_cast<int>(static_cast<long>(blockIdx.x + 1) * (rows / 128) / gridDim.x) * 128;
  const int nkc = cols / 64;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_first();
    // flat list of boxes: (tile row, kc)
    const long nbox = static_cast<long>((r1 - r0) / 128) * nkc;
    const long nst = (nbox + boxes_per_stage - 1) / boxes_per_stage;
    long issued = 0;
    unsigned long long acc = 0;
    for (long st = 0; st < nst + stages; ++st) {
      if (st >= stages) {  // consume stage st - stages
        const long c = st - stages;
        mbar_wait(&full[c % stages], static_cast<uint32_t>((c / stages) & 1));
        acc += *reinterpret_cast<volatile uint32_t*>(smem + (c % stages) * boxes_per_stage * box_bytes);
      }
      if (st < nst) {
        const int slot = static_cast<int>(st % stages);
        const int nb = static_cast<int>(min(static_cast<long>(boxes_per_stage), nbox - issued));
        mbar_expect_tx(&full[slot], nb * box_bytes);
        for (int b = 0; b < nb; ++b, ++issued) {
          const int tr = static_cast<int>(issued / nkc), kc = static_cast<int>(issued % nkc);
          tma_load_2d(smem + (slot * boxes_per_stage + b) * box_bytes, &map, &full[slot], kc * 64, r0 + tr * 128, pol);
        }
      }
    }
    if (acc == 0x12345678ull) *sink = acc;
  }
}

// 1-D variant: each CTA streams its contiguous byte range with cp.async.bulk
// (no tensor map, fully contiguous requests of `chunk` bytes).
__global__ void __launch_bounds__(64, 1)
    stream_bulk_kernel(const uint8_t* src, size_t bytes, int stages, int chunk, unsigned long long* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(stages) * chunk);
  const size_t per = (bytes / gridDim.x) & ~size_t(chunk - 1);
  const uint8_t* base = src + per * blockIdx.x;
  const long n = static_cast<long>(per / chunk);
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long acc = 0;
    for (long st = 0; st < n + stages; ++st) {
      if (st >= stages) {
        const long c = st - stages;
        mbar_wait(&full[c % stages], static_cast<uint32_t>((c / stages) & 1));
        acc += *reinterpret_cast<volatile uint32_t*>(smem + (c % stages) * chunk);
      }
      if (st < n) {
        const int slot = static_cast<int>(st % stages);
        mbar_expect_tx(&full[slot], chunk);
        bulk_load(smem + static_cast<size_t>(slot) * chunk, base + st * chunk, chunk, &full[slot]);
      }
    }
    if (acc == 0x12345678ull) *sink = acc;
  }
}

int main(int argc, char** argv) {
  const int rows = argc > 1 ? atoi(argv[1]) : 157184;
  const int cols = argc > 2 ? atoi(argv[2]) : 2048;
  void* buf;
  const size_t bytes = static_cast<size_t>(rows) * cols * 2;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  void* flushbuf;
  cudaMalloc(&flushbuf, 512u << 20);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  CUtensorMap map;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("rows=%d cols=%d bytes=%.1f MB sms=%d\n", rows, cols, bytes / 1e6, sms);
  const int configs[][2] = {{2, 1}, {3, 1}, {4, 1}, {5, 1}, {6, 1}, {8, 1}, {10, 1}, {12, 1}, {13, 1},
                            {2, 2}, {3, 2}, {4, 2}, {5, 2}, {6, 2}, {3, 4}, {2, 6}};
  for (auto& cf : configs) {
    const int stages = cf[0], bps = cf[1];
    const size_t smem = static_cast<size_t>(stages) * bps * 16384 + stages * 8 + 1024;
    if (smem > 227 * 1024) continue;
    float best = 1e9f, sum = 0.f;
    const int reps = 10;
    for (int r = 0; r < reps; ++r) {
      cudaMemsetAsync(flushbuf, r, 512u << 20);
      cudaEventRecord(e0);
      stream_kernel<<<sms, 64, smem>>>(map, rows, cols, stages, bps, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
      sum += ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("stages=%2d x %2d KB in flight=%3d KB  best %.1f us  %.0f GB/s   mean %.1f us  %.0f GB/s  %s\n", stages,
           bps * 16, stages * bps * 16, best * 1e3, bytes / (best * 1e-3) / 1e9, sum / reps * 1e3,
           bytes / (sum / reps * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  cudaFuncSetAttribute(stream_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const int bconf[][2] = {{4, 16384}, {4, 32768}, {6, 32768}, {3, 65536}, {2, 98304}};
  for (auto& cf : bconf) {
    const int stages = cf[0], chunk = cf[1];
    const size_t smem = static_cast<size_t>(stages) * chunk + stages * 8 + 1024;
    float best = 1e9f;
    for (int r = 0; r < 10; ++r) {
      cudaMemsetAsync(flushbuf, r, 512u << 20);
      cudaEventRecord(e0);
      stream_bulk_kernel<<<sms, 64, smem>>>(static_cast<const uint8_t*>(buf), bytes, stages, chunk, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    cudaError_t err = cudaGetLastError();
    printf("bulk 1-D  stages=%d x %3d KB  best %.1f us  %.0f GB/s %s\n", stages, chunk / 1024, best * 1e3,
           bytes / (best * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  // plain read kernel (LDG.128, 4 in flight per thread) for comparison
  return 0;
}
