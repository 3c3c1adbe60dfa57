// K2 smooth_mix -- the dense contraction of iteration smoothing
// (App. A.1):  Delta e_t[i] = p_t[i] W_emb, p_t = softmax(z_t).
//
// This kernel accumulates, for each position s and hidden column h,
//     acc[s, h] = sum_{v in shard} exp(f[s, v] - m_s) * E[v, h]
// relative to the rank-local max m_s (from K1's record); K3/K4 finish with
// the cross-rank rescale and the 1/l normalisation.
//
// UMMA orientation: D[h, s] (M = 128 hidden columns per sub-tile, N = positions)
//   A = E^T tile [128 h x 16 v], MN-major straight from E's row-major [V, H]
//       layout via TMA boxes of [64 h x 64 v] (no transposed copy of E);
//   B = P^T tile [N s x 16 v], K-major, produced in shared memory by 4 warps
//       from the fp32 logits: P = exp(f - m) split into bf16 hi + lo
//       (P = hi + lo to ~2^-17), two MMAs per k-step, so the bf16 operand
//       rounding stays far below the 2e-3 tolerance.
// Three rings: E tiles (HW/64 boxes per 64-v chunk, 1 KB contiguous per E row
// at HW = 512), logits chunks [N x 64] fp32 (from L2), and P tiles.  The
// logits ring runs ahead of the E ring, so an E stage is held only for its
// load and its MMAs.
// Grid: HS hidden slices x VG vocab groups (<= #SMs); each CTA writes one
// [M x HW] partial; partials are summed in fixed order downstream.
#include "common.cuh"
#include "kernels.h"

#include <cuda_bf16.h>

namespace dinfer {
namespace {

constexpr int kEpiWarps = 4;
constexpr int kThreads = (kEpiWarps + 3) * kWarpThreads;  // + E TMA, MMA, logits TMA

__host__ __device__ inline uint32_t tmem_cols_pow2(uint32_t n) {
  uint32_t c = 32;
  while (c < n) c <<= 1;
  return c;
}

struct Layout {
  uint32_t e_off, f_off, p_off, bar_off, misc_off, m_off, total;
};
__host__ __device__ inline Layout make_layout(int N, int HW, int KV, int stages, int pstages) {
  Layout L;
  const uint32_t e_stage = static_cast<uint32_t>(HW * KV) * 2u;      // HW/64 boxes of [64 h x KV v]
  const uint32_t f_stage = static_cast<uint32_t>(N * KV) * 4u;       // [N x KV] fp32
  const uint32_t p_stage = 2u * static_cast<uint32_t>(N * KV) * 2u;  // hi + lo [N x KV] bf16
  L.e_off = 0;
  L.f_off = L.e_off + static_cast<uint32_t>(stages) * e_stage;
  L.p_off = L.f_off + static_cast<uint32_t>(pstages) * f_stage;
  L.bar_off = L.p_off + static_cast<uint32_t>(pstages) * p_stage;
  L.misc_off = L.bar_off + static_cast<uint32_t>(2 * stages + 4 * pstages + 2) * 8u;
  L.m_off = L.misc_off + 16u;
  L.total = L.m_off + static_cast<uint32_t>(N) * 4u;
  return L;
}

DI uint32_t pack_bf16x2(float lo_elem, float hi_elem) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);  // .x = first (lower address)
  return *reinterpret_cast<const uint32_t*>(&v);
}

DI void advance(int& stage, uint32_t& phase, int n) {
  if (++stage == n) {
    stage = 0;
    phase ^= 1u;
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    k2_smooth_mix(const __grid_constant__ CUtensorMap map_e, const __grid_constant__ CUtensorMap map_f,
                  const K2Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const Layout L = make_layout(a.N, a.HW, a.KV, a.stages, a.pstages);
  const int warp = threadIdx.x / kWarpThreads;
  const int lane = threadIdx.x % kWarpThreads;
  const int N = a.N;
  const int KV = a.KV;                          // vocab rows per chunk: 64 (P in SW128) or 32 (SW64)
  const uint32_t ebox = 128u * static_cast<uint32_t>(KV);   // [64 h x KV v] bf16
  const uint32_t e_stage = static_cast<uint32_t>(a.HW) * 2u * static_cast<uint32_t>(KV);
  const uint32_t f_stage = static_cast<uint32_t>(N * KV) * 4u;
  const uint32_t p_row = 2u * static_cast<uint32_t>(KV);    // bytes per P row (128 or 64)
  const uint32_t p_half = static_cast<uint32_t>(N) * p_row;

  uint8_t* e_sm = smem + L.e_off;
  uint8_t* f_sm = smem + L.f_off;
  uint8_t* p_sm = smem + L.p_off;
  uint64_t* efull = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* eempty = efull + a.stages;
  uint64_t* ffull = eempty + a.stages;
  uint64_t* fempty = ffull + a.pstages;
  uint64_t* pfull = fempty + a.pstages;
  uint64_t* pempty = pfull + a.pstages;
  uint64_t* accfull = pempty + a.pstages;
  uint64_t* ready = accfull + 1;  // this CTA's vocab group of K1 slabs is complete
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + L.misc_off);
  float* m_sm = reinterpret_cast<float*>(smem + L.m_off);

  const int hs = blockIdx.x % a.HS;
  const int vg = blockIdx.x / a.HS;
  const int c0 = static_cast<int>(static_cast<long>(vg) * a.nchunks / a.VG);
  const int c1 = static_cast<int>(static_cast<long>(vg + 1) * a.nchunks / a.VG);
  const uint32_t tmem_cols = tmem_cols_pow2(static_cast<uint32_t>(a.nsub * N));

  if (a.trace != nullptr && threadIdx.x == 0) { a.trace[blockIdx.x * 5 + 0] = globaltimer_ns(); uint32_t sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm)); a.trace[blockIdx.x * 5 + 4] = sm; }
  if (warp == 4 && lane == 0) {
    prefetch_tmap(&map_e);
    prefetch_tmap(&map_f);
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&efull[i], 1);
      mbar_init(&eempty[i], 1);
    }
    for (int i = 0; i < a.pstages; ++i) {
      mbar_init(&ffull[i], 1);
      mbar_init(&fempty[i], kEpiWarps * kWarpThreads);
      mbar_init(&pfull[i], kEpiWarps * kWarpThreads);
      mbar_init(&pempty[i], 1);
    }
    mbar_init(accfull, 1);
    mbar_init(ready, 1);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(&misc[0], tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = misc[0];
  grid_dep_launch_dependents();

  if (warp == 4) {
    // ------------------------------------------------------------ TMA: E tiles
    // E does not depend on K1: streaming starts before the PDL wait, so it
    // overlaps K1's tail.
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (int c = c0; c < c1; ++c) {
        mbar_wait(&eempty[stage], phase ^ 1u);
        mbar_expect_tx(&efull[stage], e_stage);
        for (int b = 0; b < a.HW / 64; ++b)
          tma_load_2d(e_sm + stage * e_stage + b * ebox, &map_e, &efull[stage], hs * a.HW + b * 64, c * KV, pol);
        advance(stage, phase, a.stages);
      }
    }
    __syncwarp();
  } else if (warp == 6) {
    // ------------------------------------------------------------ TMA: logits chunks
    if (lane == 0) {
      // Wait for the K1 slabs of this vocab group only (not the whole K1
      // grid): their logits, partial statistics and group count are published
      // with release ordering.  The last of the HS CTAs of the group resets
      // the counters for the next step.
      const volatile unsigned* cnt = a.grp_cnt + vg;
      uint32_t spins = 0;
      while (*cnt < static_cast<unsigned>(a.SPG)) {
        __nanosleep(64);
        if (++spins > (1u << 26)) __trap();
      }
      __threadfence();
      if (atomicAdd(a.grp_pass + vg, 1u) == static_cast<unsigned>(a.HS - 1)) {
        a.grp_cnt[vg] = 0u;
        a.grp_pass[vg] = 0u;
      }
      fence_proxy_async_global();  // generic-proxy writes of K1 -> TMA reads below
      mbar_arrive(ready);
      const uint64_t pol = policy_evict_last();  // re-read by the other hidden slices
      int stage = 0;
      uint32_t phase = 0;
      for (int c = c0; c < c1; ++c) {
        mbar_wait(&fempty[stage], phase ^ 1u);
        mbar_expect_tx(&ffull[stage], f_stage);
        // f[0:N, c*64 : c*64+64]; rows >= M and columns >= V_local zero-filled
        tma_load_2d(f_sm + stage * f_stage, &map_f, &ffull[stage], c * KV, 0, pol);
        advance(stage, phase, a.pstages);
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    // warp-collective issue, per-stage descriptors advanced by constant offsets
    if (c1 > c0) {
      const uint32_t idesc = idesc_bf16(128, N, /*a MN-major*/ true, /*b K-major*/ false);
      int es = 0, ps = 0;
      uint32_t eph = 0, pph = 0;
      const int nsub = a.nsub;  // <= 8
      const uint32_t play = (KV == 64) ? 2u : 4u, psbo = 8u * p_row;  // SW128 / SW64 K-major
      for (int c = c0; c < c1; ++c) {
        mbar_wait(&pfull[ps], pph);
        mbar_wait(&efull[es], eph);
        tc_fence_after();
        if (lane == 0 && a.trace != nullptr && c == c0) a.trace[blockIdx.x * 5 + 1] = globaltimer_ns();
        // A: [128 h x 16 v] = two 64-h blocks (LBO = box bytes), 8-v groups 1 KB apart (SBO)
        const uint64_t a0 = sdesc_sw128(smem_u32(e_sm + es * e_stage), ebox, 1024);
        const uint64_t bh0 = sdesc_swz(smem_u32(p_sm + ps * 2 * p_half), 16, psbo, play);
        for (int k = 0; k < KV / 16; ++k) {
          const uint64_t bhi = sdesc_add(bh0, k * 32), blo = sdesc_add(bh0, p_half + k * 32);
#pragma unroll
          for (int sub = 0; sub < 8; ++sub) {
            if (sub < nsub) {
              const uint64_t ad = sdesc_add(a0, sub * 2 * ebox + k * 16 * 128);
              const uint32_t d = tmem_base + static_cast<uint32_t>(sub * N);
              mma_bf16_warp(d, ad, bhi, idesc, (c > c0 || k > 0) ? 1u : 0u);
              mma_bf16_warp(d, ad, blo, idesc, 1u);
            }
          }
        }
        mma_commit_warp(&eempty[es]);
        mma_commit_warp(&pempty[ps]);
        advance(es, eph, a.stages);
        advance(ps, pph, a.pstages);
      }
      mma_commit_warp(accfull);
      if (lane == 0 && a.trace != nullptr) {
        mbar_wait(accfull, 0);
        a.trace[blockIdx.x * 5 + 2] = globaltimer_ns();
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ P producers
    // Reference max of this vocab group: m_g[s] = max over its K1 slabs of the
    // partial maxima (exact max of the group's logits).  P = exp(f - m_g); the
    // partial accumulator is relative to m_g, K4 rescales with exp(m_g - m).
    const int tid = threadIdx.x;
    mbar_wait(ready, 0);
    __threadfence();
    for (int s = tid; s < N; s += kEpiWarps * kWarpThreads) {
      float mg = 0.f;
      if (s < a.M) {
        mg = neg_inf();
        const float4* ps = a.part1 + static_cast<long>(s) * a.grid1 + vg * a.SPG;
        for (int q = 0; q < a.SPG; ++q) mg = fmaxf(mg, __ldcg(&ps[q].x));
        if (hs == 0) a.mref[static_cast<long>(vg) * a.M + s] = mg;
      }
      m_sm[s] = mg;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * kWarpThreads) : "memory");
    int ps = 0;
    uint32_t pph = 0;
    for (int c = c0; c < c1; ++c) {
      mbar_wait(&ffull[ps], pph);  // logits chunk landed
      mbar_wait(&pempty[ps], pph ^ 1u);
      const float* fch = reinterpret_cast<const float*>(f_sm + ps * f_stage);
      uint8_t* phi = p_sm + ps * 2 * p_half;
      uint8_t* plo = phi + p_half;
      const int cpr = KV / 8;  // 16-B chunks per P row
      for (int u = tid; u < N * cpr; u += kEpiWarps * kWarpThreads) {
        const int s = u / cpr, cc = u - s * cpr;
        const int v0 = c * KV + cc * 8;
        float p[8];
        if (s < a.M && v0 < a.V_local) {
          const float4* src = reinterpret_cast<const float4*>(fch + s * KV + cc * 8);
          const float4 q0 = src[0], q1 = src[1];
          const float ms = m_sm[s];
          p[0] = fexp(q0.x - ms); p[1] = fexp(q0.y - ms); p[2] = fexp(q0.z - ms); p[3] = fexp(q0.w - ms);
          p[4] = fexp(q1.x - ms); p[5] = fexp(q1.y - ms); p[6] = fexp(q1.z - ms); p[7] = fexp(q1.w - ms);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) p[j] = 0.f;
        }
        float r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = p[j] - __bfloat162float(__float2bfloat16_rn(p[j]));
        const uint4 hi = make_uint4(pack_bf16x2(p[0], p[1]), pack_bf16x2(p[2], p[3]), pack_bf16x2(p[4], p[5]),
                                    pack_bf16x2(p[6], p[7]));
        const uint4 lo = make_uint4(pack_bf16x2(r[0], r[1]), pack_bf16x2(r[2], r[3]), pack_bf16x2(r[4], r[5]),
                                    pack_bf16x2(r[6], r[7]));
        // manual swizzle = the TMA/UMMA pattern: 16-B chunk index XOR address bits [7,10) (SW128) / [7,9) (SW64)
        const uint32_t swz = (KV == 64) ? (s & 7u) : ((s >> 1) & 3u);
        const uint32_t off = static_cast<uint32_t>(s) * p_row + ((static_cast<uint32_t>(cc) ^ swz) << 4);
        *reinterpret_cast<uint4*>(phi + off) = hi;
        *reinterpret_cast<uint4*>(plo + off) = lo;
      }
      mbar_arrive(&fempty[ps]);  // logits chunk consumed
      fence_proxy_async();       // generic-proxy smem writes -> visible to tcgen05.mma
      mbar_arrive(&pfull[ps]);
      advance(ps, pph, a.pstages);
    }
    // ------------------------------------------------------------ epilogue
    const int hbase = hs * a.HW;
    if (c1 > c0) {
      mbar_wait(accfull, 0);
      tc_fence_after();
    }
    // TMEM [128 h lanes x 32 s] -> smem tile [32 s][128 h] (the idle E ring)
    // -> coalesced float4 rows of the [M][H] partial.
    float* tile = reinterpret_cast<float*>(e_sm);
    for (int sub = 0; sub < a.nsub; ++sub) {
      for (int g = 0; g < N / 32; ++g) {
        float x[32];
        if (c1 > c0) {
          tmem_ld32(tmem_base + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(sub * N + g * 32), x);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) x[j] = 0.f;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) tile[j * 128 + warp * 32 + lane] = x[j];
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * kWarpThreads) : "memory");
        for (int q = threadIdx.x; q < 32 * 32; q += kEpiWarps * kWarpThreads) {
          const int row = q >> 5, c4 = q & 31;
          const int s = g * 32 + row;
          if (s < a.M)
            st_global_hint_v2(a.part + (static_cast<long>(vg) * a.M + s) * a.H + hbase + sub * 128 + c4 * 4,
                              pack_half4(*reinterpret_cast<const float4*>(tile + row * 128 + c4 * 4)),
                              policy_evict_last());
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * kWarpThreads) : "memory");
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc(tmem_base, tmem_cols);
  if (a.trace != nullptr && threadIdx.x == 0) a.trace[blockIdx.x * 5 + 3] = globaltimer_ns();
}

// Rank record finalize (vocab-sharded / split-phase path only).  Block b < M:
// one warp merges position b's K1 slab partials in a fixed order into the
// record's (m, v*, l).  Blocks >= M (when part2): rec_acc[s, h..h+3] =
// sum_g part2[g][s, h..] * e^{m_g - m_rank}, with m_rank recomputed from the
// group maxima (identical to the merged m: the groups tile the shard).
// The record is written locally (slot (epoch & 1) when double-buffered);
// with the peer exchange the last block then raises this rank's flag in every
// peer, whose K34 reads the record in place.
__global__ void rec_finalize_kernel(const RecArgs a) {
  grid_dep_wait();
  const bool need_epoch = a.par_words > 0 || a.x.peers != nullptr;
  const unsigned epoch = need_epoch ? *reinterpret_cast<volatile unsigned*>(a.x.ctl) : 0u;
  const unsigned par = epoch & 1u;
  float* rec = a.rec + (a.par_words > 0 ? par * a.par_words : 0);
  if (static_cast<int>(blockIdx.x) < a.M) {
    if (threadIdx.x < 32) {
      const int s = blockIdx.x, lane = threadIdx.x;
      float m = neg_inf(), l = 0.f;
      int ix = 0x7fffffff;
      for (int j = lane; j < a.grid1; j += 32) {
        const float4 p = __ldcg(a.part1 + static_cast<long>(s) * a.grid1 + j);
        stat_combine(m, ix, l, p.x, __float_as_int(p.y), p.z);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float rm = __shfl_xor_sync(0xffffffffu, m, o);
        const int ri = __shfl_xor_sync(0xffffffffu, ix, o);
        const float rl = __shfl_xor_sync(0xffffffffu, l, o);
        stat_combine(m, ix, l, rm, ri, rl);
      }
      if (lane == 0) {
        float* r = rec + static_cast<long>(s) * a.rec_stride;
        r[0] = m;
        r[1] = __int_as_float(ix);
        r[2] = l;
        r[3] = 0.f;
      }
    }
  } else if (a.part2 != nullptr) {
    const long t = static_cast<long>(blockIdx.x - a.M) * blockDim.x + threadIdx.x;
    const int h4 = a.H / 4;
    if (t < static_cast<long>(a.M) * h4) {
      const int s = static_cast<int>(t / h4);
      const int h = static_cast<int>(t - static_cast<long>(s) * h4) * 4;
      float mr = neg_inf();
      for (int g = 0; g < a.VG; ++g) mr = fmaxf(mr, a.mref[static_cast<long>(g) * a.M + s]);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int g = 0; g < a.VG; ++g) {
        const float sc = expf(a.mref[static_cast<long>(g) * a.M + s] - mr);
        const float4 v =
            unpack_half4(__ldcg(reinterpret_cast<const uint2*>(a.part2 + (static_cast<long>(g) * a.M + s) * a.H + h)));
        acc.x = fmaf(v.x, sc, acc.x);
        acc.y = fmaf(v.y, sc, acc.y);
        acc.z = fmaf(v.z, sc, acc.z);
        acc.w = fmaf(v.w, sc, acc.w);
      }
      *reinterpret_cast<float4*>(rec + a.acc_off + static_cast<long>(s) * a.H + h) = acc;
    }
  }
  if (a.x.peers == nullptr) return;
  // completion: every block's record writes are visible before its count; the
  // last block raises this rank's flag in every peer
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.x.ctl + 1, 1u) == gridDim.x - 1) {
      a.x.ctl[1] = 0u;
      __threadfence_system();
      for (int j = 0; j < a.x.world; ++j) {
        unsigned* f = reinterpret_cast<unsigned*>(a.x.peers[j] + a.x.flags_off) + par * a.x.world +
                      (a.x.loopback ? j : a.x.rank);
        asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch + 1u) : "memory");
      }
    }
  }
}

}  // namespace

size_t k2_smem_bytes(int N, int HW, int KV, int stages, int pstages) {
  return make_layout(N, HW, KV, stages, pstages).total + 1024;
}

cudaError_t launch_k2(const CUtensorMap& map_e, const CUtensorMap& map_f, const K2Args& a, size_t smem,
                      cudaStream_t st, bool pdl) {
  {
    const cudaError_t e = ensure_func_smem(reinterpret_cast<const void*>(k2_smooth_mix), smem);
    if (e != cudaSuccess) return e;
  }
  return launch_ex(k2_smooth_mix, dim3(a.HS * a.VG), dim3(kThreads), smem, st, pdl, map_e, map_f, a);
}

cudaError_t launch_rec_finalize(const RecArgs& a, cudaStream_t st, bool pdl) {
  const int threads = 256;
  const int acc_blocks = a.part2 == nullptr ? 0 : (a.M * (a.H / 4) + threads - 1) / threads;  // 0: stats only
  return launch_ex(rec_finalize_kernel, dim3(a.M + acc_blocks), dim3(threads), 0, st, pdl, a);
}

}  // namespace dinfer
