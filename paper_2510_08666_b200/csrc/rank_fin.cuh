// rank_fin.cuh -- the rank-record finalize folded into the tail of K12 (and
// usable by any co-resident grid): after a grid barrier, every CTA merges a
// fixed slice of the rank's record
//   stats  rec[s] = (m, v*, l) of the shard = fixed-order merge of the K1/K12
//          per-slab partials (stat_combine is exact and
//          commutative bit for bit),
//   acc    rec_acc[s, h] = sum_g part2[g][s, h] e^{m_g - m_rank}   (App. A.1,
//          the shard's share of sum_v e^{f_v - m} E[v, :]),
// and, with the peer-memory exchange, stores it straight into every rank's
// gather buffer (slot [epoch & 1][rank]); the last CTA to finish raises this
// rank's flag (epoch + 1) on every peer.  Replaces the separate record-
// finalize launch (and its serial 74-partial loop) of the sharded step.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace dinfer {

DI unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
DI void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Grid-wide barrier of a co-resident grid (checked at context creation):
// count + generation word; the last CTA to arrive resets the count and bumps
// the generation.  Consecutive uses cannot overlap: the generation is read
// before this CTA's own arrival.
DI void grid_barrier(unsigned* cnt, unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g0 = ld_acquire_gpu(gen);
    __threadfence();  // this CTA's global writes before its arrival
    if (atomicAdd(cnt, 1u) == gridDim.x - 1) {
      atomicExch(cnt, 0u);
      __threadfence();
      st_release_gpu(gen, g0 + 1u);
    } else {
      uint32_t spins = 0;
      while (ld_acquire_gpu(gen) == g0) {
        __nanosleep(32);
        if (++spins > (1u << 26)) __trap();
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Record slot of rank `a.rank` in peer j's gather buffer.  Loopback
// (measurement of one rank of a G-way shard on one GPU): every "peer" is this
// GPU's own buffer and the record is stored into all G slots, so the step
// writes the same bytes and raises the same flags a real rank would.
DI long rf_slot(const RecArgs& a, int j, unsigned par) {
  return (static_cast<long>(par) * a.world + (a.loopback ? j : a.rank)) * a.rec_words;
}
DI void rf_put(const RecArgs& a, long word, float v, unsigned par) {
  if (a.peers == nullptr) return;
  for (int j = 0; j < a.world; ++j) a.peers[j][rf_slot(a, j, par) + word] = v;
}

// The finalize proper, laid out for latency (it sits between the last K12
// CTA's partial write-out and K34 on every sharded step): after the grid
// barrier every global load a CTA needs is issued before the first one is
// used -- the statistics warp's slab partials, the acc partials of both group
// halves and the slice rows' reference maxima -- so the merge costs about one
// L2 round trip instead of one per batch.  `scratch` >= (8 + rows_max) * VG +
// 512 floats of shared memory, rows_max = ceil(elements per CTA / H) + 1 <= 8
// (checked on the host).  blockDim.x must be 256 (two group halves x 128
// float4 columns).  `tr` (DINFER_TRACE, thread 0 only): barrier passed,
// partials merged, records stored, flag raised.
constexpr int kRfLoads = 40;  // acc partial loads in flight per thread (one batch covers VG <= 80)
constexpr int kRfStat = 8;    // slab partials per lane of the statistics warp (grid1 <= 256 in one batch)

DI void rank_finalize(const RecArgs& a, unsigned* gbar, float* scratch, unsigned long long* tr) {
  grid_barrier(gbar, gbar + 1);
  if (tr != nullptr) tr[0] = globaltimer_ns();
  const unsigned epoch = (a.peers != nullptr) ? *reinterpret_cast<volatile unsigned*>(a.ctl) : 0u;
  const unsigned par = epoch & 1u;
  const int c = blockIdx.x, G1 = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ---- statistics of position c (CTA c < M, warp 7): loads issued now, merged at the end
  const bool stat_warp = c < a.M && warp == 7;
  float4 sp[kRfStat];
  if (stat_warp) {
#pragma unroll
    for (int u = 0; u < kRfStat; ++u) {
      const int j = lane + 32 * u;
      sp[u] = (j < a.grid1) ? __ldcg(a.part1 + static_cast<long>(c) * a.grid1 + j)
                            : make_float4(neg_inf(), __int_as_float(0x7fffffff), 0.f, 0.f);
    }
  }
  // ---- smoothing accumulator: CTA c owns float4 columns [q0, q1) of the flat [M][H]
  const bool has_acc = a.part2 != nullptr;
  const long nq = static_cast<long>(a.M) * a.H / 4;
  const long per = (nq + G1 - 1) / G1;
  const long q0 = static_cast<long>(c) * per, q1 = min(nq, q0 + per);
  const int half = threadIdx.x >> 7, col = threadIdx.x & 127;
  const int gh = (a.VG + 1) / 2;
  const int g0 = half * gh, g1 = min(a.VG, g0 + gh);
  const uint64_t pol = policy_evict_first();  // read once
  const int s0 = has_acc && q0 < q1 ? static_cast<int>(q0 * 4 / a.H) : 0;
  const int s1 = has_acc && q0 < q1 ? static_cast<int>((q1 * 4 - 1) / a.H) : -1;
  const int nrows = s1 - s0 + 1;
  float* mref_s = scratch;                               // [nrows][VG] group reference maxima of the rows
  float* mr = scratch + 8 * a.VG;                        // [8] m_rank of the rows
  float4* red = reinterpret_cast<float4*>(scratch + ((8 * a.VG + 8 + 3) & ~3));  // [128]
  if (has_acc && q0 < q1)
    for (int i = threadIdx.x; i < nrows * a.VG; i += blockDim.x) {
      const int r = i / a.VG, g = i - r * a.VG;
      mref_s[i] = __ldcg(a.mref + static_cast<long>(g) * a.M + s0 + r);
    }
  // column chunks of 128 float4 (one at BASELINE shapes: 111 per CTA at M = 32,
  // H = 2048); the first chunk's partial loads are issued before the maxima
  // are reduced, so the two round trips overlap
  uint2 raw[kRfLoads];
  for (long qb = q0; has_acc && qb < q1; qb += 128) {
    const long q = qb + col;
    const bool on = q < q1;
    long base = 0;
    int rr = 0;
    if (on) {
      const long e = q * 4;
      const int s = static_cast<int>(e / a.H);
      rr = s - s0;
      base = static_cast<long>(s) * a.H + (e - static_cast<long>(s) * a.H);
#pragma unroll
      for (int j = 0; j < kRfLoads; ++j)
        raw[j] = (g0 + j < g1) ? ld_global_hint_v2(a.part2 + static_cast<long>(g0 + j) * a.M * a.H + base, pol)
                               : make_uint2(0u, 0u);
    }
    if (qb == q0) {
      __syncthreads();  // mref_s
      if (warp < nrows) {  // m_rank = max over the groups' reference maxima (= the merged m)
        float m = neg_inf();
        for (int g = lane; g < a.VG; g += 32) m = fmaxf(m, mref_s[warp * a.VG + g]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) mr[warp] = m;
      }
      __syncthreads();
    }
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (on) {
      const float mrow = mr[rr];
      const float* mg = mref_s + rr * a.VG;
#pragma unroll
      for (int j = 0; j < kRfLoads; ++j) {  // fixed summation order g0, g0 + 1, ...
        if (g0 + j >= g1) break;
        const float w = __expf(mg[g0 + j] - mrow);
        const float4 v = unpack_half4(raw[j]);
        acc.x = fmaf(v.x, w, acc.x);
        acc.y = fmaf(v.y, w, acc.y);
        acc.z = fmaf(v.z, w, acc.z);
        acc.w = fmaf(v.w, w, acc.w);
      }
      for (int gb = g0 + kRfLoads; gb < g1; gb += kRfLoads) {  // VG > 2 * kRfLoads (not at BASELINE shapes)
#pragma unroll
        for (int j = 0; j < kRfLoads; ++j)
          raw[j] = (gb + j < g1) ? ld_global_hint_v2(a.part2 + static_cast<long>(gb + j) * a.M * a.H + base, pol)
                                 : make_uint2(0u, 0u);
#pragma unroll
        for (int j = 0; j < kRfLoads; ++j) {
          if (gb + j >= g1) break;
          const float w = __expf(mg[gb + j] - mrow);
          const float4 v = unpack_half4(raw[j]);
          acc.x = fmaf(v.x, w, acc.x);
          acc.y = fmaf(v.y, w, acc.y);
          acc.z = fmaf(v.z, w, acc.z);
          acc.w = fmaf(v.w, w, acc.w);
        }
      }
    }
    if (half == 1) red[col] = acc;
    __syncthreads();
    if (half == 0 && on) {
      const float4 o = red[col];
      acc.x += o.x;
      acc.y += o.y;
      acc.z += o.z;
      acc.w += o.w;
      // the record layout keeps acc 16-B aligned (stats part padded to 4 words)
      *reinterpret_cast<float4*>(a.rec_acc + base) = acc;
      if (a.peers != nullptr) {
        const long w = (a.rec_acc - a.rec) + base;
        for (int j = 0; j < a.world; ++j) *reinterpret_cast<float4*>(a.peers[j] + rf_slot(a, j, par) + w) = acc;
      }
    }
    __syncthreads();  // red reused by the next chunk
  }
  if (tr != nullptr) tr[1] = globaltimer_ns();
  if (stat_warp) {
    float m = neg_inf(), l = 0.f;
    int ix = 0x7fffffff;
#pragma unroll
    for (int u = 0; u < kRfStat; ++u)
      if (lane + 32 * u < a.grid1) stat_combine(m, ix, l, sp[u].x, __float_as_int(sp[u].y), sp[u].z);
    for (int j = lane + 32 * kRfStat; j < a.grid1; j += 32) {  // grid1 > 256 (not on B200)
      const float4 p = __ldcg(a.part1 + static_cast<long>(c) * a.grid1 + j);
      stat_combine(m, ix, l, p.x, __float_as_int(p.y), p.z);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float rm = __shfl_xor_sync(0xffffffffu, m, o);
      const int ri = __shfl_xor_sync(0xffffffffu, ix, o);
      const float rl = __shfl_xor_sync(0xffffffffu, l, o);
      stat_combine(m, ix, l, rm, ri, rl);
    }
    const long row = static_cast<long>(c) * a.rec_stride;
    if (lane == 0) {
      float* r = a.rec + row;
      r[0] = m;
      r[1] = __int_as_float(ix);
      r[2] = l;
      r[3] = 0.f;
      if (a.peers != nullptr)
        for (int j = 0; j < a.world; ++j)
          *reinterpret_cast<float4*>(a.peers[j] + rf_slot(a, j, par) + row) = make_float4(m, __int_as_float(ix), l, 0.f);
    }
    // the captured credited logits (written into the local record during the W phase)
    for (int k = lane; k < a.K && a.peers != nullptr; k += 32) rf_put(a, row + kStatWords + k, __ldcg(a.rec + row + kStatWords + k), par);
  }
  if (tr != nullptr) tr[2] = globaltimer_ns();
  if (a.peers == nullptr) return;
  // completion: this CTA's peer stores are system-visible before its count;
  // the last CTA raises this rank's flag on every peer (release)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(a.ctl + 1, 1u) == gridDim.x - 1) {
      a.ctl[1] = 0u;
      __threadfence_system();
      for (int j = 0; j < a.world; ++j) {
        unsigned* f = reinterpret_cast<unsigned*>(a.peers[j] + a.flags_off) + par * a.world + (a.loopback ? j : a.rank);
        // relaxed: the fence above orders every record store before these flags (one
        // release per flag serialised G system-scope round trips: ~2 us each)
        asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch + 1u) : "memory");
      }
    }
    if (tr != nullptr) tr[3] = globaltimer_ns();
  }
}

}  // namespace dinfer
