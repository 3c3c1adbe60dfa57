// tools/hbm_read_ceiling.cu -- calibration microbenchmark (not part of the
// product): the read-only HBM streaming ceiling of one B200, measured three
// ways so the K12 roofline is not judged against a single access pattern.
//   (1) LDG.128 (ld.global.nc.L1::no_allocate) grid-stride streams with 1..8
//       CTAs per SM, 256..1024 threads, 4..16 independent 16-B loads in flight
//       per thread;
//   (2) 2-D TMA rings of 32 KB stages (two 64-column boxes, K12's W stage
//       shape) with one CTA per SM and two CTAs per SM;
//   (3) 1-D cp.async.bulk rings.
// Every configuration reads buffers of `bytes` each, rotating over 3 buffers
// so the L2 never holds the data it reads and no dirty lines are written back
// during the timed kernel (a memset "flush" leaves ~126 MB of dirty lines that
// are written back while the next kernel reads, which lowers a read-only
// figure).  Reports best and median over reps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/hbm_read_ceiling.cu -o tools/hbm_read_ceiling
//   ./tools/hbm_read_ceiling [MB per buffer = 1288]
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2510_08666_b200/csrc/common.cuh"

using namespace dinfer;

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Each CTA reads a contiguous range (like K12's slabs); threads stride it in
// 16-B words, U loads in flight per thread.
template <int U>
__global__ void ldg_kernel(const uint4* src, size_t words, unsigned long long* sink) {
  const size_t per = (words + gridDim.x - 1) / gridDim.x;
  const size_t w0 = per * blockIdx.x, w1 = min(words, w0 + per);
  uint32_t acc = 0;
  const size_t step = static_cast<size_t>(blockDim.x) * U;
  size_t i = w0 + threadIdx.x;
  for (; i + (U - 1) * blockDim.x < w1; i += step) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_stream(src + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < w1; i += blockDim.x) {
    const uint4 v = ldg_stream(src + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9e3779b9u) *sink = acc;
}

// TMA ring: one producer thread, stages of `bps` [128 x 64] bf16 boxes (16 KB each).
// br = box rows (128: K12's W boxes; 32: its E boxes); a stage's boxes are
// adjacent 64-column chunks of one br-row tile, so a stage covers br rows x
// bps * 128 contiguous bytes per row.
__global__ void __launch_bounds__(32) tma_kernel(const __grid_constant__ CUtensorMap map, int rows, int cols, int stages,
                                                 int bps, int br, unsigned long long* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t box = 128u * static_cast<uint32_t>(br);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(stages) * bps * box);
  const int tiles = rows / br;
  const int t0 = static_cast<int>(static_cast<long>(blockIdx.x) * tiles / gridDim.x);
  const int t1 = static_cast<int>(static_cast<long>(blockIdx.x + 1) * tiles / gridDim.x);
  const int nkc = cols / 64;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
    const uint64_t pol = policy_evict_first();
    const long nbox = static_cast<long>(t1 - t0) * nkc;
    const long nst = (nbox + bps - 1) / bps;
    long issued = 0;
    unsigned long long acc = 0;
    for (long st = 0; st < nst + stages; ++st) {
      if (st >= stages) {
        const long c = st - stages;
        mbar_wait(&full[c % stages], static_cast<uint32_t>((c / stages) & 1));
        acc += *reinterpret_cast<volatile uint32_t*>(smem + (c % stages) * bps * box);
      }
      if (st < nst) {
        const int slot = static_cast<int>(st % stages);
        const int nb = static_cast<int>(min(static_cast<long>(bps), nbox - issued));
        mbar_expect_tx(&full[slot], nb * box);
        for (int b = 0; b < nb; ++b, ++issued) {
          // adjacent K chunks of one 128-row tile first (K12's 256-B-per-row stage)
          const int tr = static_cast<int>(issued / nkc), kc = static_cast<int>(issued % nkc);
          tma_load_2d(smem + (slot * bps + b) * box, &map, &full[slot], kc * 64, (t0 + tr) * br, pol);
        }
      }
    }
    if (acc == 0x12345678ull) *sink = acc;
  }
}

__global__ void __launch_bounds__(32) bulk_kernel(const uint8_t* src, size_t bytes, int stages, int chunk,
                                                  unsigned long long* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(stages) * chunk);
  const size_t per = (bytes / gridDim.x) & ~size_t(chunk - 1);
  const uint8_t* base = src + per * blockIdx.x;
  const long n = static_cast<long>(per / chunk);
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
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

// Column-blocked ("packed") W: the buffer viewed as [cols/64 column blocks]
// [rows][128 B]; each CTA owns a contiguous row slab, cut into tiles of
// `trows` rows; a stage is `cpst` adjacent column blocks of one tile, each ONE
// contiguous trows x 128 B bulk copy (K12's W stage shape from a prepacked W).
__global__ void __launch_bounds__(32) packed_kernel(const uint8_t* src, int rows, int cols, int stages, int cpst,
                                                    int trows, unsigned long long* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbytes = static_cast<uint32_t>(cpst) * trows * 128u;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(stages) * sbytes);
  const int units = rows / 32;
  const int r0 = 32 * static_cast<int>(static_cast<long>(blockIdx.x) * units / gridDim.x);
  const int r1 = 32 * static_cast<int>(static_cast<long>(blockIdx.x + 1) * units / gridDim.x);
  const int nkc = cols / 64;
  const int ntile = (r1 - r0 + trows - 1) / trows;
  const long nst = static_cast<long>(ntile) * (nkc / cpst);
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
    unsigned long long acc = 0;
    for (long st = 0; st < nst + stages; ++st) {
      if (st >= stages) {
        const long c = st - stages;
        mbar_wait(&full[c % stages], static_cast<uint32_t>((c / stages) & 1));
        acc += *reinterpret_cast<volatile uint32_t*>(smem + (c % stages) * sbytes);
      }
      if (st < nst) {
        const int slot = static_cast<int>(st % stages);
        const int t = static_cast<int>(st / (nkc / cpst)), kc0 = static_cast<int>(st % (nkc / cpst)) * cpst;
        const int row0 = r0 + t * trows, nr = min(trows, r1 - row0);
        mbar_expect_tx(&full[slot], static_cast<uint32_t>(cpst * nr * 128));
        for (int j = 0; j < cpst; ++j)
          bulk_load(smem + static_cast<size_t>(slot) * sbytes + j * trows * 128,
                    src + (static_cast<size_t>(kc0 + j) * rows + row0) * 128, nr * 128, &full[slot]);
      }
    }
    if (acc == 0x12345678ull) *sink = acc;
  }
}

struct Timer {
  cudaEvent_t e0, e1;
  Timer() {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
  }
};

template <typename F>
void measure(const char* name, size_t bytes, F launch) {
  Timer t;
  std::vector<float> ms;
  for (int r = 0; r < 3; ++r) launch(r);  // warm-up (also rotates through the buffers)
  cudaDeviceSynchronize();
  for (int r = 0; r < 12; ++r) {
    cudaEventRecord(t.e0);
    launch(r);
    cudaEventRecord(t.e1);
    cudaEventSynchronize(t.e1);
    float x;
    cudaEventElapsedTime(&x, t.e0, t.e1);
    ms.push_back(x);
  }
  cudaError_t err = cudaGetLastError();
  std::sort(ms.begin(), ms.end());
  printf("%-44s best %8.1f us %6.0f GB/s   median %8.1f us %6.0f GB/s %s\n", name, ms[0] * 1e3,
         bytes / (ms[0] * 1e-3) / 1e9, ms[ms.size() / 2] * 1e3, bytes / (ms[ms.size() / 2] * 1e-3) / 1e9,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
  fflush(stdout);
}

int main(int argc, char** argv) {
  const size_t mb = argc > 1 ? static_cast<size_t>(atol(argv[1])) : 1288;
  const int cols = 2048;
  const int rows = static_cast<int>((mb << 20) / (cols * 2) / 128 * 128);
  const size_t bytes = static_cast<size_t>(rows) * cols * 2;
  constexpr int kBufs = 3;
  void* buf[kBufs];
  for (int i = 0; i < kBufs; ++i) {
    if (cudaMalloc(&buf[i], bytes) != cudaSuccess) {
      printf("alloc failed\n");
      return 1;
    }
    cudaMemset(buf[i], i + 1, bytes);
  }
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("read ceiling: %d buffers of %.1f MB (rotated, never dirty), %d SMs\n", kBufs, bytes / 1e6, sms);

  // (1) LDG
  const int cta_per_sm[] = {1, 2, 4, 8};
  const int threads[] = {256, 512, 1024};
  for (int cps : cta_per_sm)
    for (int th : threads) {
      if (cps * th > 2048) continue;
      char name[96];
      auto run = [&](auto kern, int U) {
        snprintf(name, sizeof(name), "LDG.128 %d CTA/SM x %4d thr x %2d in flight", cps, th, U);
        measure(name, bytes, [&](int r) {
          kern<<<sms * cps, th>>>(static_cast<const uint4*>(buf[r % kBufs]), bytes / 16, sink);
        });
      };
      run(ldg_kernel<4>, 4);
      run(ldg_kernel<8>, 8);
      if (cps * th <= 1024) run(ldg_kernel<16>, 16);
    }

  // (2) TMA rings
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  CUtensorMap maps[2][kBufs];  // box rows 128 / 32
  for (int m = 0; m < 2; ++m)
    for (int i = 0; i < kBufs; ++i) {
      cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
      cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
      cuuint32_t box[2] = {64, m == 0 ? 128u : 32u}, es[2] = {1, 1};
      enc(&maps[m][i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf[i], dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  // {stages, boxes per stage, CTAs per SM, box rows}
  const int tconf[][4] = {{4, 2, 1, 128}, {5, 2, 1, 128}, {6, 2, 1, 128}, {3, 4, 1, 128}, {2, 4, 1, 128},
                          {2, 2, 2, 128}, {3, 2, 2, 128}, {2, 4, 2, 128}, {1, 6, 2, 128}, {2, 1, 4, 128},
                          {3, 1, 4, 128}, {1, 2, 4, 128},
                          {3, 16, 1, 32}, {2, 16, 1, 32}, {4, 8, 1, 32}, {6, 8, 1, 32}, {6, 4, 1, 32},
                          {12, 4, 1, 32}, {2, 32, 1, 32}, {3, 8, 2, 32}};
  for (auto& c : tconf) {
    const int stages = c[0], bps = c[1], cps = c[2], br = c[3];
    const size_t smem = static_cast<size_t>(stages) * bps * 128 * br + stages * 8 + 1024;
    if (smem * cps > 228 * 1024) continue;
    char name[96];
    snprintf(name, sizeof(name), "TMA 2-D %d CTA/SM %2d x %3d KB (%3d rows x %4d B)", cps, stages, bps * br / 8, br,
             bps * 128);
    measure(name, bytes, [&](int r) {
      tma_kernel<<<sms * cps, 32, smem>>>(maps[br == 128 ? 0 : 1][r % kBufs], rows, cols, stages, bps, br, sink);
    });
  }
  // (3) 1-D bulk
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const int bconf[][3] = {{4, 32768, 1}, {3, 65536, 1}, {2, 98304, 1}, {3, 32768, 2}, {2, 49152, 2}};
  for (auto& c : bconf) {
    const int stages = c[0], chunk = c[1], cps = c[2];
    const size_t smem = static_cast<size_t>(stages) * chunk + stages * 8 + 1024;
    char name[96];
    snprintf(name, sizeof(name), "bulk 1-D %d CTA/SM %d x %3d KB", cps, stages, chunk / 1024);
    measure(name, bytes, [&](int r) {
      bulk_kernel<<<sms * cps, 32, smem>>>(static_cast<const uint8_t*>(buf[r % kBufs]), bytes, stages, chunk, sink);
    });
  }
  // (4) packed (column-blocked) W stages
  cudaFuncSetAttribute(packed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const int pconf[][3] = {{4, 2, 160}, {4, 2, 128}, {3, 2, 160}, {5, 2, 160}, {2, 4, 160}, {4, 1, 160}};
  for (auto& c : pconf) {
    const int stages = c[0], cpst = c[1], trows = c[2];
    const size_t smem = static_cast<size_t>(stages) * cpst * trows * 128 + stages * 8 + 1024;
    if (smem > 227 * 1024) continue;
    char name[96];
    snprintf(name, sizeof(name), "packed 1 CTA/SM %d x %2d KB (%3d rows x %d blk)", stages, cpst * trows / 8, trows, cpst);
    measure(name, bytes, [&](int r) {
      packed_kernel<<<sms, 32, smem>>>(static_cast<const uint8_t*>(buf[r % kBufs]), rows, cols, stages, cpst, trows, sink);
    });
  }
  return 0;
}
