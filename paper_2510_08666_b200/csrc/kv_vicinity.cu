// Vicinity KV-cache refresh (§2.3 P:125-133,
// App. D) on a synthetic single bidirectional attention layer -- the
// KV-cache manager of Algorithm 1 (K.ShouldUpdate / K.Update).
//
// One forward (dinfer_kv_step) for block [start, end), iteration t of the block:
//   region  [lo, hi) = [0, L) while t < warmup_times or at a block's
//           completion (full refresh), else [start - prefix_look,
//           end + after_look) clipped (readings c25-c27);
//   K.Update  Kc[lo:hi] = bf16(X[lo:hi] Wk^T), Vc[lo:hi] = bf16(X[lo:hi] Wv^T)
//           -- written in place into the caller's cache; rows outside the
//           region keep their (stale) cached values;
//   queries Q = bf16(X[lo:hi] Wq^T) (the region is the forward's query region);
//   attention  out[lo:hi] = per head softmax(Q K^T / sqrt(d)) V over all L
//           cached positions (bidirectional, no mask).
// All of it runs on this file's kernels:
//   kv_proj_tc        the three projections on tcgen05 (swap-AB tiles, K split
//                     over a thread-block cluster, DSMEM reduction, bf16 rows
//                     straight into the cache / Q buffer);
//   kv_attention_tc   S = Q K^T and O = P V as tcgen05 UMMA chains per (head,
//                     128-query tile, 256-key tile), softmax from TMEM;
//   kv_attention_merge  the per-key-tile (m, l, O) partials in index order.
// The CUDA-core split-key attention (kv_attention) stays behind DINFER_KV_TC=0.
// At the steady-state region (block 32 + 2 x 16 looks = 64 queries) the layer
// is bound by the weight (3 H^2 bf16) and cache (2 L H bf16) reads.
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <new>

#include "common.cuh"
#include "dinfer.h"
#include "kernels.h"

namespace dinfer {
namespace {

constexpr int kD = 128;       // head dimension
constexpr int kQT = 64;       // queries per CTA (4 per thread row group)
constexpr int kKT = 64;       // keys per tile
constexpr int kAThreads = 256;

struct AttnArgs {
  int L, H, R, lo, nsplit, keys_per_split;
  const uint16_t* Q;   // [R][H] bf16
  const uint16_t* K;   // [L][H] bf16
  const uint16_t* V;
  float* opart;        // [nsplit][R][H]
  float* mpart;        // [nsplit][nheads][R]  (base-2 running max)
  float* lpart;
  float* out;          // [L][H] rows lo..lo+R-1
};

DI float bf2f(uint16_t u) { return __uint_as_float(static_cast<uint32_t>(u) << 16); }

constexpr size_t kAttnSmem = (kQT * kD + kD * kKT + kKT * kD + kQT * kKT + kQT * 3) * 4;

__global__ void __launch_bounds__(kAThreads) kv_attention(const AttnArgs a) {
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  float* sQ = sm;                    // [kQT][kD]   pre-scaled by log2(e)/sqrt(d)
  float* sKt = sQ + kQT * kD;        // [kD][kKT]   K tile transposed (keys contiguous)
  float* sV = sKt + kD * kKT;        // [kKT][kD]
  float* sP = sV + kKT * kD;         // [kQT][kKT]
  float* sMl = sP + kQT * kKT;       // [kQT][3]: m, l, rescale
  const int head = blockIdx.x, q0 = blockIdx.y * kQT, split = blockIdx.z;
  const int nheads = a.H / kD;
  const int tid = threadIdx.x;
  const float qscale = kLog2e * rsqrtf(static_cast<float>(kD));
  for (int e = tid; e < kQT * kD; e += kAThreads) {
    const int q = e / kD, c = e - q * kD;
    sQ[e] = (q0 + q < a.R) ? bf2f(a.Q[static_cast<long>(q0 + q) * a.H + head * kD + c]) * qscale : 0.f;
  }
  if (tid < kQT) {
    sMl[tid * 3 + 0] = neg_inf();
    sMl[tid * 3 + 1] = 0.f;
  }
  const int k_begin = split * a.keys_per_split;
  const int k_end = min(a.L, k_begin + a.keys_per_split);
  // this thread: queries 4 tq .. 4 tq + 3; keys 4 tk .. 4 tk + 3 (scores), columns 8 tk .. 8 tk + 7 (output)
  const int tq = tid / 16, tk = tid % 16;
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  for (int k0 = k_begin; k0 < k_end; k0 += kKT) {
    __syncthreads();  // previous tile consumed
    // stage K (transposed) and V tiles, bf16 -> fp32, 16-B loads of 8 columns
    for (int e = tid; e < kKT * (kD / 8); e += kAThreads) {
      const int r = e % kKT, c8 = (e / kKT) * 8;
      uint4 kv = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
      if (k0 + r < k_end) {
        const long off = static_cast<long>(k0 + r) * a.H + head * kD + c8;
        kv = __ldg(reinterpret_cast<const uint4*>(a.K + off));
        vv = __ldg(reinterpret_cast<const uint4*>(a.V + off));
      }
      const uint32_t kw[4] = {kv.x, kv.y, kv.z, kv.w}, vw[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        sKt[(c8 + 2 * u) * kKT + r] = __uint_as_float(kw[u] << 16);
        sKt[(c8 + 2 * u + 1) * kKT + r] = __uint_as_float(kw[u] & 0xffff0000u);
      }
      float4* vd = reinterpret_cast<float4*>(sV + r * kD + c8);
      vd[0] = make_float4(__uint_as_float(vw[0] << 16), __uint_as_float(vw[0] & 0xffff0000u),
                          __uint_as_float(vw[1] << 16), __uint_as_float(vw[1] & 0xffff0000u));
      vd[1] = make_float4(__uint_as_float(vw[2] << 16), __uint_as_float(vw[2] & 0xffff0000u),
                          __uint_as_float(vw[3] << 16), __uint_as_float(vw[3] & 0xffff0000u));
    }
    __syncthreads();
    // scores (base 2): a 4 x 4 register tile of Q . K * log2(e) / sqrt(d) per thread
    {
      float sc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) sc[i][j] = 0.f;
#pragma unroll 8
      for (int c = 0; c < kD; ++c) {
        const float4 kv = *reinterpret_cast<const float4*>(sKt + c * kKT + 4 * tk);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float qv = sQ[(4 * tq + i) * kD + c];
          sc[i][0] = fmaf(qv, kv.x, sc[i][0]);
          sc[i][1] = fmaf(qv, kv.y, sc[i][1]);
          sc[i][2] = fmaf(qv, kv.z, sc[i][2]);
          sc[i][3] = fmaf(qv, kv.w, sc[i][3]);
        }
      }
      const int kb = k0 + 4 * tk;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float4 s4;
        s4.x = (kb + 0 < k_end) ? sc[i][0] : neg_inf();
        s4.y = (kb + 1 < k_end) ? sc[i][1] : neg_inf();
        s4.z = (kb + 2 < k_end) ? sc[i][2] : neg_inf();
        s4.w = (kb + 3 < k_end) ? sc[i][3] : neg_inf();
        *reinterpret_cast<float4*>(sP + (4 * tq + i) * kKT + 4 * tk) = s4;
      }
    }
    __syncthreads();
    // online softmax: warp w owns query rows 8w .. 8w + 7
    {
      const int w = tid / 32, lane = tid % 32;
      for (int rr = 0; rr < kQT / 8; ++rr) {
        const int qq = (kQT / 8) * w + rr;
        const float x0 = sP[qq * kKT + lane], x1 = sP[qq * kKT + lane + 32];
        float mx = fmaxf(x0, x1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float m_old = sMl[qq * 3 + 0];
        const float m_new = fmaxf(m_old, mx);
        const float p0 = ex2(x0 - m_new), p1 = ex2(x1 - m_new);
        sP[qq * kKT + lane] = p0;
        sP[qq * kKT + lane + 32] = p1;
        float sum = p0 + p1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        __syncwarp();
        if (lane == 0) {
          const float resc = (m_old == neg_inf()) ? 0.f : ex2(m_old - m_new);
          sMl[qq * 3 + 0] = m_new;
          sMl[qq * 3 + 1] = sMl[qq * 3 + 1] * resc + sum;
          sMl[qq * 3 + 2] = resc;
        }
      }
    }
    __syncthreads();
    // O[q][c] = O[q][c] * rescale + sum_k p[q][k] V[k][c]: a 4 x 8 register tile per thread
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float resc = sMl[(4 * tq + i) * 3 + 2];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] *= resc;
    }
#pragma unroll 4
    for (int k = 0; k < kKT; ++k) {
      const float4 v0 = *reinterpret_cast<const float4*>(sV + k * kD + 8 * tk);
      const float4 v1 = *reinterpret_cast<const float4*>(sV + k * kD + 8 * tk + 4);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float p = sP[(4 * tq + i) * kKT + k];
        acc[i][0] = fmaf(p, v0.x, acc[i][0]);
        acc[i][1] = fmaf(p, v0.y, acc[i][1]);
        acc[i][2] = fmaf(p, v0.z, acc[i][2]);
        acc[i][3] = fmaf(p, v0.w, acc[i][3]);
        acc[i][4] = fmaf(p, v1.x, acc[i][4]);
        acc[i][5] = fmaf(p, v1.y, acc[i][5]);
        acc[i][6] = fmaf(p, v1.z, acc[i][6]);
        acc[i][7] = fmaf(p, v1.w, acc[i][7]);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = 4 * tq + i;
    if (q0 + q < a.R) {
      float4* o = reinterpret_cast<float4*>(a.opart + (static_cast<long>(split) * a.R + q0 + q) * a.H + head * kD +
                                            8 * tk);
      o[0] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
      o[1] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
      if (tk == 0) {
        const long mi = (static_cast<long>(split) * nheads + head) * a.R + q0 + q;
        a.mpart[mi] = sMl[q * 3 + 0];
        a.lpart[mi] = sMl[q * 3 + 1];
      }
    }
  }
}

// out[lo + r][head*128 + c..c+3] = sum_s O_s 2^{m_s - m} / sum_s l_s 2^{m_s - m}
// (splits merged in index order: deterministic), one float4 per thread.
__global__ void kv_attention_merge(const AttnArgs a) {
  grid_dep_wait();  // PDL (tcgen05 path): the key-tile partials of the attention kernel are complete
  const long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int h4 = a.H / 4;
  if (e >= static_cast<long>(a.R) * h4) return;
  const int r = static_cast<int>(e / h4), col = static_cast<int>(e - static_cast<long>(r) * h4) * 4;
  const int head = col / kD, nheads = a.H / kD;
  float m = neg_inf();
  float den = 0.f;
  float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
  constexpr int kMaxSplit = 8;
  if (a.nsplit <= kMaxSplit) {
    // every split's (m, l, O) loaded before the first use (one round trip; the
    // two-loop form below is a dependent chain of 2 x nsplit loads); the same
    // operations in the same order, so bitwise the same result
    float ms[kMaxSplit], ls[kMaxSplit];
    float4 o[kMaxSplit];
#pragma unroll
    for (int s = 0; s < kMaxSplit; ++s)
      if (s < a.nsplit) {
        const long mi = (static_cast<long>(s) * nheads + head) * a.R + r;
        ms[s] = __ldcg(a.mpart + mi);
        ls[s] = __ldcg(a.lpart + mi);
        o[s] = __ldcg(reinterpret_cast<const float4*>(a.opart + (static_cast<long>(s) * a.R + r) * a.H + col));
      }
#pragma unroll
    for (int s = 0; s < kMaxSplit; ++s)
      if (s < a.nsplit) m = fmaxf(m, ms[s]);
#pragma unroll
    for (int s = 0; s < kMaxSplit; ++s) {
      if (s >= a.nsplit || ms[s] == neg_inf()) continue;  // a split with no keys
      const float w = ex2(ms[s] - m);
      num.x = fmaf(o[s].x, w, num.x);
      num.y = fmaf(o[s].y, w, num.y);
      num.z = fmaf(o[s].z, w, num.z);
      num.w = fmaf(o[s].w, w, num.w);
      den = fmaf(ls[s], w, den);
    }
    const float inv = 1.f / den;
    *reinterpret_cast<float4*>(a.out + static_cast<long>(a.lo + r) * a.H + col) =
        make_float4(num.x * inv, num.y * inv, num.z * inv, num.w * inv);
    return;
  }
  for (int s = 0; s < a.nsplit; ++s) m = fmaxf(m, __ldcg(a.mpart + (static_cast<long>(s) * nheads + head) * a.R + r));
  for (int s = 0; s < a.nsplit; ++s) {
    const long mi = (static_cast<long>(s) * nheads + head) * a.R + r;
    const float ms = __ldcg(a.mpart + mi);
    if (ms == neg_inf()) continue;  // a split with no keys
    const float w = ex2(ms - m);
    const float4 o = __ldcg(reinterpret_cast<const float4*>(a.opart + (static_cast<long>(s) * a.R + r) * a.H + col));
    num.x = fmaf(o.x, w, num.x);
    num.y = fmaf(o.y, w, num.y);
    num.z = fmaf(o.z, w, num.z);
    num.w = fmaf(o.w, w, num.w);
    den = fmaf(__ldcg(a.lpart + mi), w, den);
  }
  const float inv = 1.f / den;
  *reinterpret_cast<float4*>(a.out + static_cast<long>(a.lo + r) * a.H + col) =
      make_float4(num.x * inv, num.y * inv, num.z * inv, num.w * inv);
}

// ---------------------------------------------------------------------------
// Tensor-core attention (tcgen05): CTA = (head, 128-query tile, kTK-key tile).
//   S = Q K^T      UMMA M=128 (queries) x N=kTK (keys) x K=128 (d), both
//                  operands K-major SW128 straight from the row-major Q / cache
//                  (TMA boxes [128|kTK rows x 64 d]); S in TMEM columns [0, kTK)
//   P = exp2((S - m) log2e / sqrt(d)) per query row (thread = row, tcgen05.ld),
//                  masked beyond L; bf16 into a K-major SW128 smem tile (the K
//                  tile's bytes, consumed by then)
//   O = P V        UMMA M=128 x N=128 (d) x K=kTK (keys): V is the MN-major B
//                  operand taken straight from the row-major cache (boxes
//                  [64 d x kTK keys], LBO between the two 64-d blocks)
// and the (m, l, O) partial of the key tile goes to the same split merge.
// ---------------------------------------------------------------------------
// 256-key tiles (80 CTAs at the steady-state region, 64 queries, L = 1088):
// 128-key tiles (144 CTAs) measured slower, 33.8 vs 32.0 us per vicinity
// forward and 132 vs 108 us per full refresh (more Q loads, 9 partials to merge)
constexpr int kTQ = 128, kTK = 256;
constexpr uint32_t kTcCols = (kTK + 128 <= 256) ? 256u : 512u;  // TMEM: S [kTK] + O [d = 128] columns
constexpr uint32_t kQBlk = kTQ * 128;    // [128 rows x 64 d] bf16 = 16 KB
constexpr uint32_t kKBlk = kTK * 128;    // [kTK rows x 64 d] bf16
constexpr uint32_t kPBlk = kTQ * 128;    // [128 q x 64 keys] bf16 = 16 KB
constexpr size_t kTcSmem = 2 * kQBlk + 2 * kKBlk + 2 * kKBlk + 64 + 1024;

struct TcArgs {
  int L, H, R, lo, nkt;
  float* opart;  // [nkt][R][H]
  float* mpart;  // [nkt][nheads][R]  base-2 max of the scaled scores
  float* lpart;
  int* cnt;      // [nheads][query tiles] key tiles done (the last one merges; self-resetting)
  float* out;    // [L][H] rows lo..lo+R-1
};

__global__ void __launch_bounds__(128, 1)
    kv_attention_tc(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                    const __grid_constant__ CUtensorMap map_v, const TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                  // 2 d-blocks
  uint8_t* sK = sQ + 2 * kQBlk;        // 2 d-blocks; reused for P (4 key-blocks of 16 KB)
  uint8_t* sV = sK + 2 * kKBlk;        // 2 d-blocks, [256 keys x 64 d] each
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + 2 * kKBlk);  // full, sdone, odone
  uint32_t* misc = reinterpret_cast<uint32_t*>(bar + 4);
  const int head = blockIdx.x, q0 = blockIdx.y * kTQ, kt = blockIdx.z, k0 = kt * kTK;
  const int nheads = a.H / kD;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    prefetch_tmap(&map_q);
    prefetch_tmap(&map_k);
    prefetch_tmap(&map_v);
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&misc[0], kTcCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = misc[0];
  const uint32_t tS = tmem, tO = tmem + kTK;
  grid_dep_launch_dependents();  // the merge kernel may launch (it waits for this grid)
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_normal();
    grid_dep_wait();  // PDL: Q and the refreshed cache rows of kv_proj_tc are complete
    // Q + K on bar[0] (S = Q K^T starts when they land), V on bar[3] (needed
    // only after the softmax)
    mbar_expect_tx(&bar[0], 2 * kQBlk + 2 * kKBlk);
    mbar_expect_tx(&bar[3], 2 * kKBlk);
    for (int j = 0; j < 2; ++j) {
      tma_load_2d(sQ + j * kQBlk, &map_q, &bar[0], head * kD + 64 * j, q0, pol);
      tma_load_2d(sK + j * kKBlk, &map_k, &bar[0], head * kD + 64 * j, k0, pol);
    }
    for (int j = 0; j < 2; ++j) tma_load_2d(sV + j * kKBlk, &map_v, &bar[3], head * kD + 64 * j, k0, pol);
    mbar_wait(&bar[0], 0);
    tc_fence_after();
    const uint32_t idesc_s = idesc_bf16(kTQ, kTK, false, false);
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_bf16(tS, sdesc_sw128(smem_u32(sQ + j * kQBlk) + k * 32, 16, 1024),
                 sdesc_sw128(smem_u32(sK + j * kKBlk) + k * 32, 16, 1024), idesc_s, (j | k) != 0);
    mma_commit(&bar[1]);
  }
  __syncwarp();
  // ---- softmax: thread = query row (TMEM lane), 256 key columns
  mbar_wait(&bar[1], 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  const uint32_t lrow = tS + (static_cast<uint32_t>(warp * 32) << 16);
  const float sc = kLog2e * rsqrtf(static_cast<float>(kD));
  float m = neg_inf();
  for (int c = 0; c < kTK / 32; ++c) {
    float x[32];
    tmem_ld32(lrow + c * 32, x);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (k0 + c * 32 + j < a.L) m = fmaxf(m, x[j]);
  }
  const float ms = m * sc;  // base-2 max of the scaled scores
  float l = 0.f;
  for (int c = 0; c < kTK / 32; ++c) {
    float x[32];
    tmem_ld32(lrow + c * 32, x);
    uint32_t pk[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int kk = k0 + c * 32 + 2 * j;
      const float p0 = (kk < a.L) ? ex2(fmaf(x[2 * j], sc, -ms)) : 0.f;
      const float p1 = (kk + 1 < a.L) ? ex2(fmaf(x[2 * j + 1], sc, -ms)) : 0.f;
      l += p0 + p1;
      const __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
      pk[j] = *reinterpret_cast<const uint32_t*>(&b2);
    }
    // keys c*32 .. c*32+31 -> key block (c / 2), 16-B chunks ((c % 2) * 4 + u) of this row, SW128
    uint8_t* blk = sK + (c / 2) * kPBlk + row * 128;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t chunk = static_cast<uint32_t>((c % 2) * 4 + u) ^ static_cast<uint32_t>(row & 7);
      *reinterpret_cast<uint4*>(blk + chunk * 16) = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
    }
  }
  fence_proxy_async();  // P (generic smem writes) -> visible to tcgen05.mma
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    // O[128 q x 128 d] = P[128 q x 256 keys] V[256 keys x 128 d]; V MN-major:
    // 128-B rows of 64 d per key, 8-key atoms 1 KB apart (SBO), the two 64-d
    // blocks kKBlk apart (LBO)
    const uint32_t idesc_o = idesc_bf16(kTQ, kD, false, /*b MN-major*/ true);
    mbar_wait(&bar[3], 0);  // V landed
    tc_fence_after();
#pragma unroll
    for (int kb = 0; kb < kTK / 64; ++kb)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_bf16(tO, sdesc_sw128(smem_u32(sK + kb * kPBlk) + k * 32, 16, 1024),
                 sdesc_sw128(smem_u32(sV) + (kb * 64 + k * 16) * 128, kKBlk, 1024), idesc_o, (kb | k) != 0);
    mma_commit(&bar[2]);
  }
  __syncwarp();
  mbar_wait(&bar[2], 0);
  tc_fence_after();
  const uint32_t orow = tO + (static_cast<uint32_t>(warp * 32) << 16);
  const bool valid = q0 + row < a.R;
  float* op = a.opart + (static_cast<long>(kt) * a.R + q0 + row) * a.H + head * kD;
  for (int c = 0; c < kD / 32; ++c) {
    float x[32];
    tmem_ld32(orow + c * 32, x);
    if (valid) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(op + c * 32 + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
    }
  }
  if (valid) {
    const long mi = (static_cast<long>(kt) * nheads + head) * a.R + q0 + row;
    a.mpart[mi] = ms;
    a.lpart[mi] = l;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, kTcCols);
}

// ---------------------------------------------------------------------------
// K.Update + queries on tcgen05 (`kv_proj_tc`): Y_m[p, :] = bf16(X[p, :] W_m^T)
// for the three projections m = K, V, Q over the refresh region's positions.
// Swap-AB tiles: D[128 output features x NT positions] = W_m[f-tile, :] X[p-tile, :]^T,
// both operands K-major SW128 straight from the row-major weights / layer
// input (TMA boxes [128 | NT rows x 64 k]), fp32 accumulator in TMEM.  At the
// steady-state region (64 positions) the 3 H^2 weights are the only real
// traffic (HBM-bound, AI = 64 flop/B), so the H-deep contraction is split
// over a thread-block cluster of `ks` CTAs along K (grid = 3 H/128 tiles x ks
// ~ one CTA per SM); the partial accumulators are reduced in the leader CTA
// through distributed shared memory in rank order (deterministic), and the
// leader writes bf16 rows of 16-B chunks into the cache / Q buffer.
// ---------------------------------------------------------------------------
constexpr int kPjMaxStages = 8;             // ring depth cap of the measurement override
constexpr uint32_t kPjWBox = 128u * 128u;  // [128 rows x 64 k] bf16

struct ProjArgs {
  int H, R, lo, NT, nkc, ks, stages, cps;  // cps: 64-wide K chunks per ring stage
  uint16_t* dst[3];   // row p of projection m at dst[m] + (p - dst_row0[m]) * H
  int dst_row0[3];
};

// The ring, or (if larger) the epilogue's [NT][128] fp32 tile + bf16 rows that
// reuse it; the barriers follow.
__host__ __device__ inline size_t kv_proj_body(int NT, int stages, int cps) {
  const size_t ring = static_cast<size_t>(stages) * cps * (kPjWBox + static_cast<uint32_t>(NT) * 128u);
  const size_t epi = static_cast<size_t>(NT) * 128u * 6u;
  return ring > epi ? ring : epi;
}
__host__ __device__ inline size_t kv_proj_smem(int NT, int stages, int cps) {
  return kv_proj_body(NT, stages, cps) + 2 * stages * 8 + 64 + 1024;
}

DI uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
DI void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 16 B of CTA `rank`'s shared memory at this CTA's address `local_addr`
// (distributed shared memory); no completion wait, so several can be in flight.
DI float4 ld_dsmem_v4(const void* local_addr, uint32_t rank) {
  uint32_t a = smem_u32(local_addr), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(r));
  return v;
}

__global__ void __launch_bounds__(128, 1)
    kv_proj_tc(const __grid_constant__ CUtensorMap map_w0, const __grid_constant__ CUtensorMap map_w1,
               const __grid_constant__ CUtensorMap map_w2, const __grid_constant__ CUtensorMap map_x, const ProjArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t xbox = static_cast<uint32_t>(a.NT) * 128u;
  const int cps = a.cps;
  const uint32_t slot = static_cast<uint32_t>(cps) * (kPjWBox + xbox);  // [cps W boxes][cps X boxes]
  const uint32_t xoff = static_cast<uint32_t>(cps) * kPjWBox;
  const int nst = a.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kv_proj_body(a.NT, nst, cps));
  uint64_t* empty = full + nst;
  uint64_t* done = empty + nst;
  uint32_t* misc = reinterpret_cast<uint32_t*>(done + 1);
  const int ftiles = a.H / 128;
  const int m = blockIdx.x / ftiles, ft = blockIdx.x - m * ftiles;
  const int p0 = a.lo + blockIdx.y * a.NT;
  const int z = static_cast<int>(blockIdx.z);
  const int kc0 = z * a.nkc / a.ks, kc1 = (z + 1) * a.nkc / a.ks;
  const CUtensorMap* mw = (m == 0) ? &map_w0 : (m == 1) ? &map_w1 : &map_w2;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    prefetch_tmap(mw);
    prefetch_tmap(&map_x);
    for (int i = 0; i < nst; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&misc[0], 256);
  grid_dep_launch_dependents();  // the attention kernel may launch (it waits for this grid)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = misc[0];
  if (threadIdx.x == 0) {  // TMA producer
    const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
    for (int kc = kc0, i = 0; kc < kc1; kc += cps, ++i) {
      const int st = i % nst, nc = min(cps, kc1 - kc);
      if (i >= nst) mbar_wait(&empty[st], static_cast<uint32_t>((i / nst - 1) & 1));
      uint8_t* sl = smem + st * slot;
      mbar_expect_tx(&full[st], static_cast<uint32_t>(nc) * (kPjWBox + xbox));
      for (int j = 0; j < nc; ++j) {
        tma_load_2d(sl + j * kPjWBox, mw, &full[st], (kc + j) * 64, ft * 128, pol_w);
        tma_load_2d(sl + xoff + j * xbox, &map_x, &full[st], (kc + j) * 64, p0, pol_x);  // rows past L: zero fill
      }
    }
  } else if (warp == 1) {  // MMA issuer (warp-collective issue, common.cuh mma_bf16_warp)
    const uint32_t idesc = idesc_bf16(128, a.NT, false, false);
    for (int kc = kc0, i = 0; kc < kc1; kc += cps, ++i) {
      const int st = i % nst, nc = min(cps, kc1 - kc);
      mbar_wait(&full[st], static_cast<uint32_t>((i / nst) & 1));
      tc_fence_after();
      for (int j = 0; j < nc; ++j) {
        const uint64_t da = sdesc_sw128(smem_u32(smem + st * slot + j * kPjWBox), 16, 1024);
        const uint64_t db = sdesc_sw128(smem_u32(smem + st * slot + xoff + j * xbox), 16, 1024);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_bf16_warp(tmem, sdesc_add(da, k * 32), sdesc_add(db, k * 32), idesc, (i | j | k) != 0 ? 1u : 0u);
      }
      mma_commit_warp(&empty[st]);
    }
    mma_commit_warp(done);
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();
  // ---- epilogue: thread = output feature (TMEM lane); columns = positions
  float* red = reinterpret_cast<float*>(smem);  // [NT][128] fp32 (the idle ring)
  const uint32_t lrow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  const int feat = threadIdx.x;
  const bool split = a.ks > 1;
  for (int c0 = 0; c0 < a.NT; c0 += 32) {
    float x[32];
    tmem_ld32(lrow + c0, x);
#pragma unroll
    for (int j = 0; j < 32; ++j) red[(c0 + j) * 128 + feat] = x[j];
  }
  tc_fence_before();
  if (split) cluster_sync_all();  // every CTA's partial in its shared memory
  else __syncthreads();
  // Every CTA of the cluster finishes 1/ks of the tile's positions: the ks
  // partials summed in rank order ((p0 + p1) + p2, whichever CTA sums --
  // bitwise the leader-only epilogue this replaces), bf16, 8-B stores of 4
  // features (a warp covers a position's 256-B row segment).  The leader-only
  // version left the other CTAs parked at the final cluster barrier (~45 % of
  // the kernel's stall samples, ncu).
  const int rank = split ? static_cast<int>(cluster_ctarank()) : 0, nr = split ? a.ks : 1;
  const int q_lo = (rank * a.NT / nr) * 32, q_hi = ((rank + 1) * a.NT / nr) * 32;
  uint16_t* dst = (m == 0) ? a.dst[0] : (m == 1) ? a.dst[1] : a.dst[2];  // no dynamic param indexing
  const int row0 = (m == 0) ? a.dst_row0[0] : (m == 1) ? a.dst_row0[1] : a.dst_row0[2];
  const float4* red4 = reinterpret_cast<const float4*>(red);
  for (int q0 = q_lo + static_cast<int>(threadIdx.x); q0 < q_hi; q0 += 4 * 128) {
    float4 v[4][4];  // [u][rank]: 4 x ks loads in flight
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int q = q0 + u * 128;
        if (r < nr && q < q_hi) v[u][r] = (r == rank) ? red4[q] : ld_dsmem_v4(red4 + q, static_cast<uint32_t>(r));
      }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = q0 + u * 128;
      if (q >= q_hi) continue;
      float4 acc = v[u][0];
#pragma unroll
      for (int r = 1; r < 4; ++r)
        if (r < nr) {
          acc.x += v[u][r].x;
          acc.y += v[u][r].y;
          acc.z += v[u][r].z;
          acc.w += v[u][r].w;
        }
      const int c = q / 32, f4 = q % 32, pos = p0 + c;
      if (pos < a.lo + a.R) {
        const __nv_bfloat162 b01 = __floats2bfloat162_rn(acc.x, acc.y), b23 = __floats2bfloat162_rn(acc.z, acc.w);
        uint2 w;
        w.x = *reinterpret_cast<const uint32_t*>(&b01);
        w.y = *reinterpret_cast<const uint32_t*>(&b23);
        *reinterpret_cast<uint2*>(dst + static_cast<long>(pos - row0) * a.H + ft * 128 + f4 * 4) = w;
      }
    }
  }
  if (split) cluster_sync_all();  // every CTA's shared memory stays valid until its peers have read it
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 256);
}

PFN_cuTensorMapEncodeTiled_v12000 kv_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// [outer][inner] bf16 row-major, SWIZZLE_128B boxes [box_outer][64]
bool kv_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_outer) {
  auto fn = kv_encoder();
  if (fn == nullptr) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace
}  // namespace dinfer

using namespace dinfer;

struct dinfer_kv {
  dinfer_kv_shape shp{};
  cudaStream_t stream = nullptr;
  int num_sms = 0;
  size_t smem_optin = 0;  // per-block opt-in shared memory (kv_proj_tc ring depth)
  // kv_proj_tc ring: 4 stages of one 64-wide K chunk (same-box A/B at the MoE
  // attention shape, tools/kv_ab.sh: 33.1-33.2 us per vicinity forward vs
  // 33.4 for 2 x 2 chunks, 33.7 for 3 x 1, 35.0 for 2 x 1, 42.0 for 3 x 2 --
  // footprints that leave one CTA per SM strand clusters of ks CTAs in a second
  // wave); env DINFER_KV_PJ_STAGES / DINFER_KV_PJ_CPS (measurement)
  int pj_stages = 4;
  int pj_nt = 0, pj_ks = 0, pj_st = 0;  // cached ring depth for (NT, ks)
  int pj_cps = 1;  // K chunks per kv_proj_tc stage, at most
  int pj_cur_cps = 1;
  bool pdl = true;               // PDL between the projections, the attention and the merge (env DINFER_KV_PDL)
  int ks_max = 4;                // kv_proj_tc cluster split of K cap (env DINFER_KV_KS, measurement)
  uint16_t* Q = nullptr;  // [L][H]
  float* opart = nullptr;
  float* mpart = nullptr;
  float* lpart = nullptr;
  size_t part_rows = 0;   // capacity of opart in rows of H
  bool tc = true;         // tcgen05 attention (DINFER_KV_TC=0: the CUDA-core kernel)
  CUtensorMap map_q{}, map_k{}, map_v{};
  const void* c_k = nullptr;
  const void* c_v = nullptr;
  int* cnt = nullptr;          // [nheads][query tiles] merge counters
  // projection maps (kv_proj_tc), cached per pointer / per position-tile width
  CUtensorMap map_wq{}, map_wk{}, map_wv{}, map_x{};
  const void* c_wq = nullptr;
  const void* c_wk = nullptr;
  const void* c_wv = nullptr;
  const void* c_x = nullptr;
  int c_xnt = 0;
};

extern "C" {

int32_t dinfer_kv_region(const dinfer_kv_shape* s, int32_t start, int32_t end, int32_t t, int32_t full,
                         int32_t* lo, int32_t* hi) {
  if (s == nullptr || lo == nullptr || hi == nullptr) return -1;
  if (full || t < s->warmup_times) {
    *lo = 0;
    *hi = s->L;
  } else {
    *lo = std::max(0, start - s->prefix_look);
    *hi = std::min(s->L, end + s->after_look);
  }
  return *hi - *lo;
}

dinfer_status dinfer_kv_create(const dinfer_kv_shape* s, void* stream, dinfer_kv** out) {
  if (s == nullptr || out == nullptr) return DINFER_ERR_ARG;
  *out = nullptr;
  if (s->L < 1 || s->H < kD || s->H % kD != 0 || s->d_head != kD) return DINFER_ERR_SHAPE;
  if (s->prefix_look < 0 || s->after_look < 0 || s->warmup_times < 0) return DINFER_ERR_ARG;
  dinfer_kv* c = new (std::nothrow) dinfer_kv();
  if (c == nullptr) return DINFER_ERR_NOMEM;
  c->shp = *s;
  c->stream = static_cast<cudaStream_t>(stream);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t LH = static_cast<size_t>(s->L) * s->H;
  // split partials: CUDA-core kernel <= 4 L rows; tcgen05 kernel one per 256-key tile
  c->part_rows = std::max(static_cast<size_t>(s->L) * 4 + 256,
                          static_cast<size_t>((s->L + kTK - 1) / kTK) * static_cast<size_t>(s->L));
  const size_t nml = c->part_rows * (s->H / kD);
  bool ok = cudaMalloc(&c->Q, LH * 2) == cudaSuccess && cudaMalloc(&c->opart, c->part_rows * s->H * 4) == cudaSuccess &&
            cudaMalloc(&c->mpart, nml * 4) == cudaSuccess && cudaMalloc(&c->lpart, nml * 4) == cudaSuccess;
  const size_t ncnt = static_cast<size_t>(s->H / kD) * ((s->L + kTQ - 1) / kTQ);
  if (ok) ok = cudaMalloc(&c->cnt, ncnt * 4) == cudaSuccess && cudaMemset(c->cnt, 0, ncnt * 4) == cudaSuccess;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  c->smem_optin = optin > 0 ? static_cast<size_t>(optin) : kv_proj_smem(256, 2, 1);
  if (ok) ok = ensure_func_smem(reinterpret_cast<const void*>(kv_proj_tc), c->smem_optin) == cudaSuccess;
  if (const char* e = std::getenv("DINFER_KV_TC")) c->tc = std::atoi(e) != 0;
  if (const char* e = std::getenv("DINFER_KV_PDL")) c->pdl = std::atoi(e) != 0;
  if (const char* e = std::getenv("DINFER_KV_PJ_CPS")) c->pj_cps = std::max(1, std::min(4, std::atoi(e)));
  if (const char* e = std::getenv("DINFER_KV_KS")) c->ks_max = std::max(1, std::min(8, std::atoi(e)));
  if (const char* e = std::getenv("DINFER_KV_PJ_STAGES")) c->pj_stages = std::max(2, std::min(kPjMaxStages, std::atoi(e)));
  if (ok && c->tc) {
    ok = kv_map(&c->map_q, c->Q, static_cast<uint64_t>(s->H), static_cast<uint64_t>(s->L), kTQ) &&
         cudaFuncSetAttribute(kv_attention_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(kTcSmem)) == cudaSuccess;
  }
  if (ok) ok = cudaFuncSetAttribute(kv_attention, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kAttnSmem)) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    dinfer_kv_destroy(c);
    return DINFER_ERR_NOMEM;
  }
  *out = c;
  return DINFER_OK;
}

void dinfer_kv_destroy(dinfer_kv* c) {
  if (c == nullptr) return;
  if (c->stream != nullptr) cudaStreamSynchronize(c->stream);
  cudaFree(c->Q);
  cudaFree(c->opart);
  cudaFree(c->mpart);
  cudaFree(c->lpart);
  cudaFree(c->cnt);
  delete c;
}

dinfer_status dinfer_kv_step(dinfer_kv* c, const uint16_t* X, const uint16_t* Wq, const uint16_t* Wk,
                             const uint16_t* Wv, uint16_t* Kc, uint16_t* Vc, int32_t start, int32_t end, int32_t t,
                             int32_t full, float* out, int32_t* lo_hi) {
  if (c == nullptr || X == nullptr || Wq == nullptr || Wk == nullptr || Wv == nullptr || Kc == nullptr ||
      Vc == nullptr || out == nullptr)
    return DINFER_ERR_ARG;
  const int L = c->shp.L, H = c->shp.H;
  if (start < 0 || end <= start || end > L || t < 0) return DINFER_ERR_ARG;
  for (const void* p : {static_cast<const void*>(X), static_cast<const void*>(Kc), static_cast<const void*>(Vc)})
    if (reinterpret_cast<uintptr_t>(p) % 16 != 0) return DINFER_ERR_SHAPE;
  int32_t lo = 0, hi = 0;
  const int R = dinfer_kv_region(&c->shp, start, end, t, full, &lo, &hi);
  if (lo_hi != nullptr) {
    lo_hi[0] = lo;
    lo_hi[1] = hi;
  }
  // ---- K.Update + queries: Y_m[R, H] = bf16(X[lo:hi] W_m^T), m = K, V, Q, on
  // tcgen05 (kv_proj_tc): K / V straight into the cache rows, Q into c->Q
  {
    auto wmap = [&](CUtensorMap* mp, const void** cache, const uint16_t* Wp) {
      if (*cache == Wp) return true;
      if (!kv_map(mp, Wp, static_cast<uint64_t>(H), static_cast<uint64_t>(H), 128)) return false;
      *cache = Wp;
      return true;
    };
    if (!wmap(&c->map_wk, &c->c_wk, Wk) || !wmap(&c->map_wv, &c->c_wv, Wv) || !wmap(&c->map_wq, &c->c_wq, Wq))
      return DINFER_ERR_CUDA;
    // position tiles of NT <= 256 (multiple of 16), then split K over a
    // cluster of up to 4 CTAs while the grid is under one CTA per SM
    const int ntp = (R + 255) / 256;
    const int NT = ((R + ntp - 1) / ntp + 15) / 16 * 16;
    if (X != c->c_x || NT != c->c_xnt) {
      if (!kv_map(&c->map_x, X, static_cast<uint64_t>(H), static_cast<uint64_t>(L), static_cast<uint32_t>(NT)))
        return DINFER_ERR_CUDA;
      c->c_x = X;
      c->c_xnt = NT;
    }
    const int tiles = 3 * (H / 128) * ntp, nkc = H / 64;
    const int ks = std::max(1, std::min({c->ks_max, std::max(1, c->ks_max > 4 ? 2 * c->num_sms / tiles : c->num_sms / tiles), nkc}));
    ProjArgs pa{};
    pa.H = H;
    pa.R = R;
    pa.lo = lo;
    pa.NT = NT;
    pa.nkc = nkc;
    pa.ks = ks;
    // Ring geometry: stages of cps K chunks, the deepest ring (<= pj_stages)
    // that fits (DINFER_KV_PJ_CPS / DINFER_KV_PJ_STAGES; defaults measured,
    // see kv_create)
    if (c->pj_nt != NT || c->pj_ks != ks) {
      c->pj_cur_cps = c->pj_cps;
      c->pj_st = 0;
      for (int cps = c->pj_cps; cps >= 1 && c->pj_st == 0; --cps)
        for (int st = c->pj_stages; st >= 2; --st)
          if (kv_proj_smem(NT, st, cps) <= c->smem_optin) {
            c->pj_st = st;
            c->pj_cur_cps = cps;
            break;
          }
      if (c->pj_st == 0) return DINFER_ERR_UNSUPPORTED;
      c->pj_nt = NT;
      c->pj_ks = ks;
    }
    pa.stages = c->pj_st;
    pa.cps = c->pj_cur_cps;
    pa.dst[0] = Kc;
    pa.dst[1] = Vc;
    pa.dst[2] = c->Q;
    pa.dst_row0[0] = 0;
    pa.dst_row0[1] = 0;
    pa.dst_row0[2] = lo;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(3 * (H / 128), ntp, ks);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = kv_proj_smem(NT, pa.stages, pa.cps);
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = static_cast<unsigned>(ks);
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kv_proj_tc, c->map_wk, c->map_wv, c->map_wq, c->map_x, pa) != cudaSuccess)
      return DINFER_ERR_CUDA;
  }
  // ---- attention over all L cached positions
  if (c->tc) {
    if (Kc != c->c_k) {
      if (!kv_map(&c->map_k, Kc, H, L, kTK)) return DINFER_ERR_CUDA;
      c->c_k = Kc;
    }
    if (Vc != c->c_v) {
      if (!kv_map(&c->map_v, Vc, H, L, kTK)) return DINFER_ERR_CUDA;
      c->c_v = Vc;
    }
    const int nh = H / kD, nkt = (L + kTK - 1) / kTK, nqt = (R + kTQ - 1) / kTQ;
    if (static_cast<size_t>(nkt) * R > c->part_rows) return DINFER_ERR_SHAPE;
    TcArgs t{};
    t.L = L;
    t.H = H;
    t.R = R;
    t.lo = lo;
    t.nkt = nkt;
    t.opart = c->opart;
    t.mpart = c->mpart;
    t.lpart = c->lpart;
    t.cnt = c->cnt;
    t.out = out;
    // PDL chain: the attention CTAs launch while the projections drain (setup,
    // TMEM allocation) and wait for them before their loads; the merge likewise
    if (launch_ex(kv_attention_tc, dim3(nh, nqt, nkt), dim3(128), kTcSmem, c->stream, c->pdl, c->map_q, c->map_k,
                  c->map_v, t) != cudaSuccess)
      return DINFER_ERR_CUDA;
    AttnArgs m{};
    m.L = L;
    m.H = H;
    m.R = R;
    m.lo = lo;
    m.nsplit = nkt;
    m.opart = c->opart;
    m.mpart = c->mpart;
    m.lpart = c->lpart;
    m.out = out;
    const long n4 = static_cast<long>(R) * H / 4;
    if (launch_ex(kv_attention_merge, dim3(static_cast<unsigned>((n4 + 127) / 128)), dim3(128), 0, c->stream, c->pdl,
                  m) != cudaSuccess)
      return DINFER_ERR_CUDA;
    return DINFER_OK;
  }
  const int nheads = H / kD, qtiles = (R + kQT - 1) / kQT;
  // about one CTA per SM: each split re-reads the query tile and writes a partial
  int nsplit = std::max(1, (c->num_sms + nheads * qtiles - 1) / (nheads * qtiles));
  nsplit = std::min(nsplit, std::max(1, (L + kKT - 1) / kKT));
  while (static_cast<size_t>(nsplit) * R > c->part_rows && nsplit > 1) --nsplit;
  const int kps = (((L + nsplit - 1) / nsplit + kKT - 1) / kKT) * kKT;
  nsplit = (L + kps - 1) / kps;
  AttnArgs a{};
  a.L = L;
  a.H = H;
  a.R = R;
  a.lo = lo;
  a.nsplit = nsplit;
  a.keys_per_split = kps;
  a.Q = c->Q;
  a.K = Kc;
  a.V = Vc;
  a.opart = c->opart;
  a.mpart = c->mpart;
  a.lpart = c->lpart;
  a.out = out;
  kv_attention<<<dim3(nheads, qtiles, nsplit), kAThreads, kAttnSmem, c->stream>>>(a);
  const long n4 = static_cast<long>(R) * H / 4;
  kv_attention_merge<<<static_cast<unsigned>((n4 + 127) / 128), 128, 0, c->stream>>>(a);
  if (cudaGetLastError() != cudaSuccess) return DINFER_ERR_CUDA;
  return DINFER_OK;
}

}  // extern "C"
