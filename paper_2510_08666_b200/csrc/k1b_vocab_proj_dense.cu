// K1b vocab_proj_dense -- the compute-bound regime of the LM-head contraction
// + softmax statistics for many positions
// (M > 256, e.g. LLaDA-8B bs64 x block 64 = 4096 positions, BASELINE
// configs[4]).  Normal orientation: positions on UMMA M, vocab on N.
//
//   logits[s, v] = h[s, :] . W[v, :]
//
// Work unit = (256-position block, vocab group); the grid is persistent over
// units.  Per unit the CTA walks the group's 256-wide vocab blocks; per block
// it streams K = H in 64-wide chunks: A = hidden rows [256 x 64] (two 128-row
// TMA boxes), B = W rows [256 x 64]; two tcgen05.mma 128x256x16 per k-step
// (one per 128-position half) into two 256-column fp32 TMEM accumulators
// (the whole 512-column TMEM), 128 flop per byte of L2 traffic.
// Epilogue (4 warps, lane = position): tcgen05.ld 32 columns at a time and a
// per-thread online softmax (chunk max, one rescale, 32 exps) -- no cross-lane
// reduction at all in this orientation.  At the end of a unit each position's
// (m, v*, l) over the vocab group is written as one "record" row, so K3
// combines vocab groups exactly like vocab-sharded ranks.
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace dinfer {
namespace {

constexpr int kEpiWarps = 4;
constexpr int kThreads = (kEpiWarps + 2) * kWarpThreads;
constexpr int kBM = 256;                              // positions per unit
constexpr int kBN = 256;                              // vocab columns per block
constexpr uint32_t kBox = 128u * 128u;                // [128 rows x 64 k] bf16 = 16 KB
constexpr uint32_t kStageBytes = 4u * kBox;           // A 2 boxes + B 2 boxes = 64 KB
constexpr uint32_t kTmemCols = 512;

struct Layout {
  uint32_t st_off, bar_off, misc_off, total;
};
__host__ __device__ inline Layout make_layout(int stages) {
  Layout L;
  L.st_off = 0;
  L.bar_off = static_cast<uint32_t>(stages) * kStageBytes;
  L.misc_off = L.bar_off + static_cast<uint32_t>(2 * stages + 2) * 8u;
  L.total = L.misc_off + 16u;
  return L;
}

DI void advance(int& stage, uint32_t& phase, int n) {
  if (++stage == n) {
    stage = 0;
    phase ^= 1u;
  }
}

// Online softmax statistics of 32 new logits (ids id0 .. id0+31, `nvalid`
// of them valid) into the running (m, idx, l) of one position.
DI void online32(const float (&x)[32], int id0, int nvalid, float& m, int& idx, float& l) {
  float cm = neg_inf();
  int ci = INT_MAX;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const bool ok = j < nvalid;
    if (ok && x[j] > cm) {  // strict: first (lowest id) maximum within the chunk
      cm = x[j];
      ci = id0 + j;
    }
  }
  if (nvalid <= 0) return;
  const float mn = fmaxf(m, cm);
  const float mref = mn * kLog2e;
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) s += (j < nvalid) ? ex2(fmaf(x[j], kLog2e, -mref)) : 0.f;
  l = (m == neg_inf() ? 0.f : l * ex2(fmaf(m, kLog2e, -mref))) + s;
  if (cm > m) idx = ci;  // ties with an earlier (lower-id) chunk keep the earlier id
  m = mn;
}

__global__ void __launch_bounds__(kThreads, 1)
    k1b_vocab_proj_dense(const __grid_constant__ CUtensorMap map_h, const __grid_constant__ CUtensorMap map_w,
                         const K1bArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const Layout L = make_layout(a.stages);
  const int warp = threadIdx.x / kWarpThreads;
  const int lane = threadIdx.x % kWarpThreads;
  uint8_t* st_sm = smem + L.st_off;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty = full + a.stages;
  uint64_t* tfull = empty + a.stages;
  uint64_t* tempty = tfull + 1;
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + L.misc_off);

  const int nmb = (a.M + kBM - 1) / kBM;
  const int nunits = nmb * a.VG;
  const int nkc = a.H / kKChunk;
  const int nblocks = (a.V_local + kBN - 1) / kBN;

  if (warp == 4 && lane == 0) {
    prefetch_tmap(&map_h);
    prefetch_tmap(&map_w);
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, kEpiWarps * kWarpThreads);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(&misc[0], kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = misc[0];
  grid_dep_launch_dependents();

  // units in vocab-group-major order: the position blocks of one vocab group
  // run concurrently and share each W block through L2
  auto unit_coords = [&](int u, int& mb, int& g) {
    g = u / nmb;
    mb = u - g * nmb;
  };
  auto block_range = [&](int g, int& b0, int& b1) {
    b0 = static_cast<int>(static_cast<long>(g) * nblocks / a.VG);
    b1 = static_cast<int>(static_cast<long>(g + 1) * nblocks / a.VG);
  };

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      grid_dep_wait();
      const uint64_t pol_h = policy_evict_last();   // hidden blocks re-read by every vocab group
      const uint64_t pol_w = policy_evict_normal();  // W blocks re-read by the position blocks of a group
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        int mb, g, b0, b1;
        unit_coords(u, mb, g);
        block_range(g, b0, b1);
        for (int nb = b0; nb < b1; ++nb) {
          for (int kc = 0; kc < nkc; ++kc) {
            mbar_wait(&empty[stage], phase ^ 1u);
            mbar_expect_tx(&full[stage], kStageBytes);
            uint8_t* dst = st_sm + stage * kStageBytes;
            tma_load_2d(dst, &map_h, &full[stage], kc * kKChunk, mb * kBM, pol_h);
            tma_load_2d(dst + kBox, &map_h, &full[stage], kc * kKChunk, mb * kBM + 128, pol_h);
            tma_load_2d(dst + 2 * kBox, &map_w, &full[stage], kc * kKChunk, nb * kBN, pol_w);
            tma_load_2d(dst + 3 * kBox, &map_w, &full[stage], kc * kKChunk, nb * kBN + 128, pol_w);
            advance(stage, phase, a.stages);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    // warp-collective issue, per-stage descriptors advanced by constant offsets
    const uint32_t idesc = idesc_bf16(128, kBN, false, false);
    int stage = 0;
    uint32_t phase = 0, tuse = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      int mb, g, b0, b1;
      unit_coords(u, mb, g);
      block_range(g, b0, b1);
      for (int nb = b0; nb < b1; ++nb) {
        mbar_wait(tempty, (tuse & 1u) ^ 1u);  // epilogue drained both accumulators
        tc_fence_after();
        for (int kc = 0; kc < nkc; ++kc) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          // B = W rows [256 x 16]: two 128-row boxes 16 KB apart = rows 8..255 at SBO 1 KB,
          // so one descriptor spans both boxes (box 1 follows box 0 contiguously)
          const uint64_t d0 = sdesc_sw128(smem_u32(st_sm + stage * kStageBytes), 16, 1024);
#pragma unroll
          for (int k = 0; k < kKChunk / 16; ++k) {
            const uint32_t acc = (kc | k) != 0;
            const uint64_t bd = sdesc_add(d0, 2 * kBox + k * 32);
            mma_bf16_warp(tmem_base, sdesc_add(d0, k * 32), bd, idesc, acc);
            mma_bf16_warp(tmem_base + kBN, sdesc_add(d0, kBox + k * 32), bd, idesc, acc);
          }
          mma_commit_warp(&empty[stage]);
          advance(stage, phase, a.stages);
        }
        mma_commit_warp(tfull);
        ++tuse;
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    uint32_t tuse = 0;
    const int r = warp * 32 + lane;  // TMEM lane = position within each 128-half
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      int mb, g, b0, b1;
      unit_coords(u, mb, g);
      block_range(g, b0, b1);
      float m0 = neg_inf(), l0 = 0.f, m1 = neg_inf(), l1 = 0.f;
      int i0 = INT_MAX, i1 = INT_MAX;
      for (int nb = b0; nb < b1; ++nb) {
        mbar_wait(tfull, tuse & 1u);
        tc_fence_after();
        const int nvalid_blk = min(kBN, a.V_local - nb * kBN);
#pragma unroll 1
        for (int c = 0; c < kBN / 32; ++c) {
          float x0[32], x1[32];
          const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
          tmem_ld32(tmem_base + lane_off + static_cast<uint32_t>(c * 32), x0);
          tmem_ld32(tmem_base + lane_off + static_cast<uint32_t>(kBN + c * 32), x1);
          if (c == kBN / 32 - 1) {  // both accumulators fully read: MMA may overwrite
            tc_fence_before();
            mbar_arrive(tempty);
          }
          const int id0 = a.v_offset + nb * kBN + c * 32;
          const int nv = nvalid_blk - c * 32;
          online32(x0, id0, nv, m0, i0, l0);
          online32(x1, id0, nv, m1, i1, l1);
        }
        ++tuse;
      }
      // one record row per position of this unit: (m, v*, l, 0) for vocab group g
      const int s0 = mb * kBM + r, s1 = mb * kBM + 128 + r;
      float4* out = reinterpret_cast<float4*>(a.part) + static_cast<long>(g) * a.M;
      if (s0 < a.M) out[s0] = make_float4(m0, __int_as_float(i0), l0, 0.f);
      if (s1 < a.M) out[s1] = make_float4(m1, __int_as_float(i1), l1, 0.f);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc(tmem_base, kTmemCols);
}

}  // namespace

size_t k1b_smem_bytes(int stages) { return make_layout(stages).total + 1024; }

cudaError_t launch_k1b(const CUtensorMap& map_h, const CUtensorMap& map_w, const K1bArgs& a, int grid, size_t smem,
                       cudaStream_t st, bool pdl) {
  {
    const cudaError_t e = ensure_func_smem(reinterpret_cast<const void*>(k1b_vocab_proj_dense), smem);
    if (e != cudaSuccess) return e;
  }
  return launch_ex(k1b_vocab_proj_dense, dim3(grid), dim3(kThreads), smem, st, pdl, map_h, map_w, a);
}

}  // namespace dinfer
