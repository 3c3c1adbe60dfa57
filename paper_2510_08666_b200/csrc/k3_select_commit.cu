// K3 select_commit -- combine the per-rank statistics, credit update + fuse,
// threshold / hierarchical selection, commit.  K4 smooth_finalize -- the
// iteration-smoothing output e_{t+1} for positions still masked.
//
// K3: kSelPos (16) positions per CTA, the last CTA of a batch row to finish
// phase 1 runs phase 2 for the row.  Phase 1 is warp-per-position / lane-per-slot:
//   combine   m = max_r m_r, v* = v*_r of the maximiser (lowest id on ties),
//             l = sum_r l_r e^{m_r - m} in rank order; lse = m + ln l; p* = 1/l
//
//   credit    undecided rows: C <- beta*C; C[v*] += p*^gamma  (Eq. credit-update,
//             P:306-313) on K sparse slots (exactly the dense table: untouched
//             tokens have C = 0); hit / first-empty slot found by warp ballots;
//             fuse f~ = f + alpha ln(1+C) (Eq. logits-fuse); only
//             credited tokens change, so
//             lse~ = m + ln(l + sum_{cred} e^{f_v - m}((1+C_v)^alpha - 1)),
//             v~ = argmax_{cred u {v*}} f~ (lowest id on ties), p~ = e^{f~_{v~} - lse~}
//             (warp-shuffle reductions in a fixed order).
// Phase 2 is thread-per-position:
//   select    threshold (strict '>' or '>=' with params.inclusive,
//             fallback max) or hierarchical
//             (maximal runs of undecided positions; per run the
//             best position, ties nearest the run centre then lower index,
//             if p~ > theta_lo), via ballots and shared-memory atomics.
//   commit    tokens[s] = v~, mask[s] = 0, committed[s] = 1
// K4: e_{t+1}[s,:] = e_mask + alpha_t * (sum_p acc_p[s,:] e^{m_p - m}) / l
//     for rows still undecided (App. A.1).
#include <algorithm>
#include <climits>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

#include <cuda_bf16.h>

namespace dinfer {
namespace {

constexpr int kMaxS = 1024;
// 512 threads: the kernel needs ~110 registers (1024 threads would cap it at
// 64 and spill to local memory, each spill a dependent L1/L2 round trip)
constexpr int kK3Threads = 512;
constexpr int kPer = kMaxS / kK3Threads;  // positions per thread in the selection

DI int run_first(const uint32_t* words, int s) {
  int w = s >> 5;
  uint32_t z = ~words[w] & ((1u << (s & 31)) - 1u);  // non-region bits below s
  while (z == 0u) {
    if (--w < 0) return 0;
    z = ~words[w];
  }
  return (w << 5) + (31 - __clz(z)) + 1;
}
DI int run_last(const uint32_t* words, int s, int nwords) {
  int w = s >> 5;
  const int b = s & 31;
  uint32_t z = (b == 31) ? 0u : (~words[w] & ~((2u << b) - 1u));  // non-region bits above s
  while (z == 0u) {
    if (++w >= nwords) return (nwords << 5) - 1;
    z = ~words[w];
  }
  return (w << 5) + __ffs(z) - 2;
}

// argmax with the lowest id on ties, over (value, id) pairs of a warp
DI void warp_argmax(float& v, int& id) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, id, o);
    if (ov > v || (ov == v && oi < id)) {
      v = ov;
      id = oi;
    }
  }
}
DI float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Credit update (Eq. credit-update) on the K <= 32 slots of one
// undecided position, slot k in lane k (warp-collective): every credited slot
// decays by beta, then v*'s slot gains p*^gamma (or v* claims the first empty
// slot).  Returns true if v* had no slot and none was free.  Shared by the
// selection blocks and (credit-fused smoothing) the smoothing blocks, so both
// see bit-identical credit values.
DI bool credit_update_slots(float beta, float gamma, bool slot, int vstar, float pstar, int& cid, float& cv) {
  const float gain = ex2(gamma * __log2f(pstar));  // p*^gamma
  if (cid >= 0) cv = beta * cv;
  const int lane = threadIdx.x & 31;
  const unsigned hb = __ballot_sync(0xffffffffu, slot && cid == vstar);
  const unsigned eb = __ballot_sync(0xffffffffu, slot && cid < 0);
  const int hit = hb ? __ffs(hb) - 1 : -1, empty = eb ? __ffs(eb) - 1 : -1;
  if (hit >= 0) {
    if (lane == hit) cv += gain;
  } else if (empty >= 0) {
    if (lane == empty) {
      cid = vstar;
      cv = gain;
    }
  }
  return hit < 0 && empty < 0;
}

// Fuse of one credited slot (Eq. logits-fuse): ft = f_k + alpha
// ln(1 + C_k) (f_k = m for v*, else the captured raw logit fc); returns the
// slot's share of the fused partition function relative to e^m,
// w_k = e^{f_k - m}((1 + C_k)^alpha - 1) (non-credited tokens are unchanged).
DI float credit_fuse_slot(float alpha, int cid, float cv, int vstar, float m, float fc, float& ft) {
  const float fk = (cid == vstar) ? m : fc;
  const float lc = __logf(1.f + cv);
  ft = fk + alpha * lc;
  return __expf(fk - m) * (__expf(alpha * lc) - 1.f);
}

// Warp-collective: merged statistics (m, v*, l) of position i, from K1's
// per-slab partials (single rank) or from the `world` records (rank order).
// Every lane returns the identical, deterministic result.  Split into the
// loads (issued ahead, see select_block) and the merge.
constexpr int kStatU = 5;  // slab partials per lane in one round trip (grid1 <= 160)
struct StatIn {
  float4 p[kStatU];
};
DI void stats_load(const K3Args& a, int i, int lane, StatIn& q) {
  if (a.part1 != nullptr) {
    const float4* src = a.part1 + static_cast<long>(i) * a.grid1;
#pragma unroll
    for (int u = 0; u < kStatU; ++u) {
      const int j = lane + 32 * u;
      q.p[u] = (j < a.grid1) ? __ldcg(src + j) : make_float4(neg_inf(), __int_as_float(INT_MAX), 0.f, 0.f);
    }
    return;
  }
  q.p[0] = (lane < a.world) ? *reinterpret_cast<const float4*>(a.rb[lane] + static_cast<long>(i) * a.rec_stride)
                            : make_float4(neg_inf(), __int_as_float(INT_MAX), 0.f, 0.f);
}
DI void stats_merge(const K3Args& a, int i, int lane, const StatIn& q, float& m, int& vstar, float& l) {
  m = neg_inf();
  l = 0.f;
  vstar = INT_MAX;
  if (a.part1 != nullptr) {
    // lanes stride the slabs, then an xor butterfly (stat_combine is
    // commutative bit for bit, so all lanes agree)
#pragma unroll
    for (int u = 0; u < kStatU; ++u) stat_combine(m, vstar, l, q.p[u].x, __float_as_int(q.p[u].y), q.p[u].z);
    for (int j = lane + 32 * kStatU; j < a.grid1; j += 32) {  // grid1 > 160 (not on B200)
      const float4 p = __ldcg(a.part1 + static_cast<long>(i) * a.grid1 + j);
      stat_combine(m, vstar, l, p.x, __float_as_int(p.y), p.z);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float rm = __shfl_xor_sync(0xffffffffu, m, o);
      const int rv = __shfl_xor_sync(0xffffffffu, vstar, o);
      const float rl = __shfl_xor_sync(0xffffffffu, l, o);
      stat_combine(m, vstar, l, rm, rv, rl);
    }
    return;
  }
  m = q.p[0].x;
  vstar = __float_as_int(q.p[0].y);
  l = q.p[0].z;
  float m0 = m, l0 = l;  // merge ranks 1..world-1 into lane 0 in rank order, then broadcast
  int v0 = vstar;
  for (int r = 1; r < a.world; ++r) {
    const float mr = __shfl_sync(0xffffffffu, m, r);
    const int vr = __shfl_sync(0xffffffffu, vstar, r);
    const float lr = __shfl_sync(0xffffffffu, l, r);
    stat_combine(m0, v0, l0, mr, vr, lr);
  }
  m = __shfl_sync(0xffffffffu, m0, 0);
  vstar = __shfl_sync(0xffffffffu, v0, 0);
  l = __shfl_sync(0xffffffffu, l0, 0);
}
DI void row_stats(const K3Args& a, int i, int lane, float& m, int& vstar, float& l) {
  StatIn q;
  stats_load(a, i, lane, q);
  stats_merge(a, i, lane, q, m, vstar, l);
}

// Per-position inputs of phase 1, loaded one position ahead of their use.
struct PosIn {
  StatIn st;
  int cid;
  float cv, fc;
  bool und;
};
DI void pos_load(const K3Args& a, int i, int lane, PosIn& q) {
  const long roff = static_cast<long>(i) * a.rec_stride;
  const long cbase = static_cast<long>(i) * a.K;
  q.und = a.block_start || a.mask[i] != 0;  // block start: every position undecided
  const bool slot = a.use_credit && a.K <= 32 && lane < a.K;  // slot k in lane k, kept in registers
  q.cid = (slot && !a.block_start) ? a.credit_ids[cbase + lane] : -1;  // block start: slots empty
  q.cv = (slot && !a.block_start) ? a.credit_val[cbase + lane] : 0.f;
  q.fc = 0.f;  // raw logit of the credited token (max over ranks: -inf where not owned)
  if (slot) {
    q.fc = a.rb[0][roff + kStatWords + lane];
    for (int r = 1; r < a.world; ++r) q.fc = fmaxf(q.fc, a.rb[r][roff + kStatWords + lane]);
  }
  stats_load(a, i, lane, q.st);
}

// Selection CTAs: phase 1 covers kSelPos positions per CTA, each warp a strided subset
// of them with the next position's loads issued before the current one is
// processed (the per-position chain is latency-bound: one round trip per
// warp instead of one per position).  With S > kSelPos each CTA writes its
// positions' (p~, v~, undecided) to `sel`, and the last CTA of the row to
// arrive (counter, release/acquire fences) runs phase 2 over the whole row.
// 16 positions per selection CTA (two CTAs per 32-position block, the last to
// arrive runs phase 2): phase 1 one position per warp.  Same-box A/B against 32:
// MoE step 214.0-214.2 vs 214.9-215.0 us, V/8 rank 62.4-62.6 vs 63.3-63.5 us.
#ifndef DINFER_SEL_POS
#define DINFER_SEL_POS 16
#endif
constexpr int kSelPos = DINFER_SEL_POS;
// smoothing blocks: 128 float4 columns x 4 partial groups (512 consecutive elements; one
// wave of <= 144 blocks at the MoE shape)
constexpr int kSmCols = 128, kSmGroups = 4, kSmBatch = 8;
#ifndef DINFER_SM_HB
#define DINFER_SM_HB 20
#endif
constexpr int kSmBatchH = DINFER_SM_HB;  // fp16 partial loads in flight per thread (74 partials / 4 groups in one round trip)
DI int sel_ctas_per_row(int S) { return (S + kSelPos - 1) / kSelPos; }

DI void select_block(const K3Args& a, int c, unsigned long long* tr) {
  __shared__ uint32_t s_reg[kMaxS / 32];
  __shared__ int s_runA[kMaxS];
  __shared__ unsigned long long s_runkey[kMaxS];
  __shared__ float s_pt[kMaxS];
  __shared__ int s_vt[kMaxS];
  __shared__ uint8_t s_und[kMaxS];
  __shared__ unsigned long long s_best;
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int cps = sel_ctas_per_row(a.S);
  const int b = c / cps, chunk = c - b * cps;

  // ------------------------------------------------------------ phase 1
  const int s_end = min(a.S, (chunk + 1) * kSelPos);
  PosIn nxt;
  if (chunk * kSelPos + warp < s_end) pos_load(a, b * a.S + chunk * kSelPos + warp, lane, nxt);
  for (int s = chunk * kSelPos + warp; s < s_end; s += nwarps) {
    const PosIn cur = nxt;
    if (s + nwarps < s_end) pos_load(a, b * a.S + s + nwarps, lane, nxt);  // the next position, ahead
    const int i = b * a.S + s;
    const long roff = static_cast<long>(i) * a.rec_stride;
    const long cbase = static_cast<long>(i) * a.K;
    const bool und = cur.und;
    const bool fast = a.use_credit && a.K <= 32;  // slot k in lane k, kept in registers
    const bool slot = fast && lane < a.K;
    int cid = cur.cid;
    float cv = cur.cv;
    // device-checked precondition (SPEC: a credit entry is never negative; ids
    // index the vocabulary): sticky flag, surfaced by dinfer_sync
    if (und && slot && cid >= 0 && (cid >= a.V_total || !(cv >= 0.f))) atomicOr(a.err, kErrCreditInvalid);
    const float fc = cur.fc;
    float m, l;
    int vstar;
    stats_merge(a, i, lane, cur.st, m, vstar, l);
    const float lse = m + __logf(l);
    const float pstar = __frcp_rn(l);  // == 1.0f / l (correctly rounded), no slow path
    int vt = vstar;
    float pt = pstar;
    if (fast && und) {
      if (credit_update_slots(a.c_beta, a.c_gamma, slot, vstar, pstar, cid, cv) && lane == 0)
        atomicOr(a.err, kErrCreditSlotsFull);
      if (slot) {
        a.credit_ids[cbase + lane] = cid;
        a.credit_val[cbase + lane] = cv;
      }
      // fuse over credited tokens (v* included)
      float best = m, extra = 0.f;
      int best_id = vstar;
      if (cid >= 0) {
        float ft;
        extra = credit_fuse_slot(a.c_alpha, cid, cv, vstar, m, fc, ft);
        if (ft > best || (ft == best && cid < best_id)) {
          best = ft;
          best_id = cid;
        }
      }
      extra = warp_sum(extra);
      warp_argmax(best, best_id);
      const float lse_t = m + __logf(l + extra);
      vt = best_id;
      pt = __expf(best - lse_t);
    } else if (a.use_credit && und) {  // K > 32: slots strided over the lanes
      if (a.block_start) {  // slots empty before this step's update
        for (int k = lane; k < a.K; k += 32) {
          a.credit_ids[cbase + k] = -1;
          a.credit_val[cbase + k] = 0.f;
        }
        __syncwarp();
      }
      const float gain = ex2(a.c_gamma * __log2f(pstar));  // p*^gamma
      // pass 1: decay, locate the slot of v* (or the first empty one)
      int hit = -1, empty = -1;
      for (int k0 = 0; k0 < a.K; k0 += 32) {
        const int k = k0 + lane;
        const int id = (k < a.K) ? a.credit_ids[cbase + k] : INT_MAX;
        if (k < a.K && id >= 0) {
          const float cv0 = a.credit_val[cbase + k];
          if (id >= a.V_total || !(cv0 >= 0.f)) atomicOr(a.err, kErrCreditInvalid);
          a.credit_val[cbase + k] = a.c_beta * cv0;
        }
        const unsigned hb = __ballot_sync(0xffffffffu, k < a.K && id == vstar);
        const unsigned eb = __ballot_sync(0xffffffffu, k < a.K && id < 0);
        if (hit < 0 && hb) hit = k0 + __ffs(hb) - 1;
        if (empty < 0 && eb) empty = k0 + __ffs(eb) - 1;
      }
      __syncwarp();  // decayed values visible to lane 0
      if (lane == 0) {
        if (hit >= 0) {
          a.credit_val[cbase + hit] += gain;
        } else if (empty >= 0) {
          a.credit_ids[cbase + empty] = vstar;
          a.credit_val[cbase + empty] = gain;
        } else {
          atomicOr(a.err, kErrCreditSlotsFull);
        }
      }
      __syncwarp();
      // pass 2: fuse over credited tokens (v* included)
      float best = m, extra = 0.f;
      int best_id = vstar;
      for (int k0 = 0; k0 < a.K; k0 += 32) {
        const int k = k0 + lane;
        const int id = (k < a.K) ? a.credit_ids[cbase + k] : -1;
        if (id >= 0) {
          float fk = m;
          if (id != vstar) {
            fk = a.rb[0][roff + kStatWords + k];
            for (int r = 1; r < a.world; ++r) fk = fmaxf(fk, a.rb[r][roff + kStatWords + k]);
          }
          const float lc = __logf(1.f + a.credit_val[cbase + k]);
          const float ft = fk + a.c_alpha * lc;
          extra += __expf(fk - m) * (__expf(a.c_alpha * lc) - 1.f);
          if (ft > best || (ft == best && id < best_id)) {
            best = ft;
            best_id = id;
          }
        }
      }
      extra = warp_sum(extra);
      warp_argmax(best, best_id);
      const float lse_t = m + __logf(l + extra);
      vt = best_id;
      pt = __expf(best - lse_t);
    }
    if (lane == 0) {
      if (a.stats != nullptr) {
        float* st = a.stats + static_cast<long>(i) * 4;
        st[0] = m;
        st[1] = lse;
        st[2] = pt;
        st[3] = __int_as_float(vt);
      }
      a.ml[2 * i] = m;
      a.ml[2 * i + 1] = l;
      if (cps == 1) {
        s_pt[s] = pt;
        s_vt[s] = vt;
        s_und[s] = und ? 1 : 0;
      } else {
        a.sel[i] = make_float4(pt, __int_as_float(vt), und ? 1.f : 0.f, 0.f);
        __threadfence();  // release: this position before the arrival below
      }
    }
  }
  if (cps > 1) {  // last CTA of the row to arrive runs phase 2
    __syncthreads();
    if (threadIdx.x == 0) {
      const int prev = atomicAdd(a.row_cnt + b, 1);
      s_last = prev == cps - 1;
      if (s_last) {
        __threadfence();  // acquire: the other CTAs' positions
        a.row_cnt[b] = 0;  // all arrived: reset for the next step
      }
    }
    __syncthreads();
    if (!s_last) {
      if (tr != nullptr) tr[2] = globaltimer_ns();
      return;
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int s = threadIdx.x + q * kK3Threads;
      if (s < a.S) {
        const float4 v = __ldcg(a.sel + static_cast<long>(b) * a.S + s);
        s_pt[s] = v.x;
        s_vt[s] = __float_as_int(v.y);
        s_und[s] = v.z != 0.f;
      }
    }
  }
  __syncthreads();
  if (tr != nullptr) tr[2] = globaltimer_ns();

  // ------------------------------------------------------------ phase 2: selection
  // position s = threadIdx.x + q * kK3Threads (q < kPer); its ballot word is warp + q * nwarps
  const int nwords = (a.S + 31) / 32;
  const float thr_primary = (a.decoder == 0) ? a.tau : a.theta_hi;
  // reading c1: "exceeds" is strict; variant c1' (params.inclusive) is SPEC's '>='
  const bool incl = a.inclusive != 0;
  auto clears = [incl](float p, float thr) { return incl ? p >= thr : p > thr; };
  bool A[kPer], und[kPer], region[kPer];
  float pt[kPer];
  int first[kPer];
  unsigned long long key[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int s = threadIdx.x + q * kK3Threads;
    const bool valid = s < a.S;
    und[q] = valid && s_und[s];
    pt[q] = valid ? s_pt[s] : 0.f;
    A[q] = und[q] && clears(pt[q], thr_primary);
    region[q] = false;
    first[q] = 0;
    key[q] = 0ull;
  }
  if (a.decoder == 1) {
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int s = threadIdx.x + q * kK3Threads;
      region[q] = und[q] && !(a.runs_after_hi && A[q]);
      const unsigned rb = __ballot_sync(0xffffffffu, region[q]);
      if (lane == 0 && warp + q * nwarps < nwords) s_reg[warp + q * nwarps] = rb;
      if (s < a.S) {
        s_runA[s] = 0;
        s_runkey[s] = 0ull;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      if (!region[q]) continue;
      const int s = threadIdx.x + q * kK3Threads;
      first[q] = run_first(s_reg, s);
      const int last = run_last(s_reg, s, nwords);
      if (A[q]) atomicOr(&s_runA[first[q]], 1);
      const int dist = abs(2 * s - first[q] - last);
      key[q] = (static_cast<unsigned long long>(__float_as_uint(pt[q])) << 32) |
               (static_cast<unsigned long long>(0xFFFF - dist) << 16) | static_cast<unsigned long long>(0xFFFF - s);
      atomicMax(&s_runkey[first[q]], key[q]);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kPer; ++q)
      if (region[q] && !s_runA[first[q]] && s_runkey[first[q]] == key[q] && clears(pt[q], a.theta_lo)) A[q] = true;
  }
  if (threadIdx.x == 0) s_best = 0ull;
  bool mine = false;
#pragma unroll
  for (int q = 0; q < kPer; ++q) mine = mine || A[q];
  const int anyA = __syncthreads_or(mine);
  if (!anyA) {  // fallback: the undecided position with max p~ (lowest index on ties)
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int s = threadIdx.x + q * kK3Threads;
      if (und[q])
        atomicMax(&s_best, (static_cast<unsigned long long>(__float_as_uint(pt[q])) << 32) |
                               static_cast<unsigned long long>(0xFFFFFFFFu - s));
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int s = threadIdx.x + q * kK3Threads;
      A[q] = und[q] && s_best != 0ull &&
             static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(s_best & 0xFFFFFFFFull)) == s;
    }
  }

  // ------------------------------------------------------------ commit
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int s = threadIdx.x + q * kK3Threads;
    if (s < a.S) {
      const int i = b * a.S + s;
      a.committed[i] = A[q] ? 1 : 0;
      s_und[s] = A[q] ? 1 : 0;  // reused below: committed by this step
      if (A[q]) {
        a.tokens[i] = s_vt[s];
        a.mask[i] = 0;
      } else if (a.block_start) {  // the block's state is written whole
        a.tokens[i] = a.mask_id;
        a.mask[i] = 1;
      }
    }
  }
  if (a.emb == nullptr) return;
  // ------------------------------------------------------------ next-iteration input embedding (f2)
  // The smoothing blocks wrote every row of this batch row (E[token] for rows
  // decided at step start, bf16(e_{t+1}) for the others); once all of them
  // have counted in, the rows committed by this step are overwritten with
  // their new token's embedding row E[v~] (smoothing feeds only
  // positions that stay masked).
  constexpr int kSmElems = kSmCols * 4;
  for (int s = threadIdx.x; s < a.S; s += blockDim.x) {
    const long i = static_cast<long>(b) * a.S + s;
    const int need = static_cast<int>(((i + 1) * a.H - 1) / kSmElems - (i * a.H) / kSmElems + 1);
    const volatile int* cnt = a.rowdone + i;
    uint32_t spins = 0;
    while (*cnt < need) {
      __nanosleep(32);
      if (++spins > (1u << 26)) __trap();
    }
  }
  __syncthreads();
  __threadfence();
  const int h8 = a.H / 8;
  for (int u = threadIdx.x; u < a.S * h8; u += blockDim.x) {
    const int s = u / h8, c8 = u - s * h8;
    if (s_und[s]) {
      const long i = static_cast<long>(b) * a.S + s;
      *reinterpret_cast<uint4*>(a.emb + i * a.H + c8 * 8) =
          *reinterpret_cast<const uint4*>(a.E + static_cast<long>(s_vt[s]) * a.H + c8 * 8);
    }
  }
  for (int s = threadIdx.x; s < a.S; s += blockDim.x) a.rowdone[static_cast<long>(b) * a.S + s] = 0;
}

// Smoothing block: 512 threads = 128 float4 columns x 4 partial groups, i.e.
// 512 consecutive elements of the [M, H] output.  Each thread accumulates a
// strided subset of the nparts partials (online rescale, overlapping the
// statistics merge), the 4 groups are combined in a fixed order through
// shared memory (deterministic).  The block merges the statistics (m, l) of
// the rows it covers itself (one warp per row), so it does not wait for the
// selection; rows undecided at step START are written (e_{t+1} matters for
// those still undecided after the commit).
// Partials p = grp, grp + kSmGroups, ... of element (s, h..h+3), all loads of
// a round issued before any use, merged relative to the round's max M of the
// partial maxima: pacc = sum_p e^{m_p - M} acc_p (fixed order; a later round,
// only for nparts > kB * kSmGroups, rescales the running sum).  Two passes over
// registers, no data-dependent branches: the online-rescale form this replaces
// was ~2 K SASS instructions of K34's i-cache-bound smoothing path (ncu:
// 35 % of K34's stall samples "no instruction").
template <int kB, bool kHalf>
DI void accumulate_parts(const K4Args& a, int s, int h, int grp, float4& pacc, float& mrun) {
  static_assert(kHalf, "fp32 partials arrive as rank records (accumulate_recs)");
  const uint64_t pol = policy_evict_first();  // read once
  const long step = static_cast<long>(kSmGroups) * a.acc_stride;
  const uint16_t* src = a.acc_h + static_cast<long>(s) * a.H + h + grp * a.acc_stride;
  const float* msrc = a.m_part + grp * a.m_stride + static_cast<long>(s) * a.m_rowstride;
  const long mstep = static_cast<long>(kSmGroups) * a.m_stride;
  for (int p0 = grp; p0 < a.nparts; p0 += kB * kSmGroups) {
    uint2 raw[kB];
    float mp[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      const bool ok = p0 + j * kSmGroups < a.nparts;
      raw[j] = ok ? ld_global_hint_v2(src + j * step, pol) : make_uint2(0u, 0u);
      mp[j] = ok ? msrc[j * mstep] : neg_inf();
    }
    src += kB * step;
    msrc += kB * mstep;
    float M = mrun;
#pragma unroll
    for (int j = 0; j < kB; ++j) M = fmaxf(M, mp[j]);
    if (M == neg_inf()) continue;  // no partial in this round (or all empty)
    if (mrun != neg_inf() && M != mrun) {
      const float r = __expf(mrun - M);
      pacc.x *= r;
      pacc.y *= r;
      pacc.z *= r;
      pacc.w *= r;
    }
    mrun = M;
#pragma unroll
    for (int j = 0; j < kB; ++j) {  // fixed summation order; an empty partial (m = -inf) adds exactly 0
      const bool live = mp[j] != neg_inf();
      const float4 vj = unpack_half4(live ? raw[j] : make_uint2(0u, 0u));
      const float sc = live ? __expf(mp[j] - M) : 0.f;
      pacc.x = fmaf(vj.x, sc, pacc.x);
      pacc.y = fmaf(vj.y, sc, pacc.y);
      pacc.z = fmaf(vj.z, sc, pacc.z);
      pacc.w = fmaf(vj.w, sc, pacc.w);
    }
  }
}

// The world rank records in rank order (K12 record mode / sharded steps):
// pacc = sum_r e^{m_r - mrun} acc_r with the online rescale to the running max
// (m_r = record r's merged max); all loads issued before the first use.
// rec_unit (world 1, K12 record mode): the one record is relative to the
// merged m itself -- taken as is (scale 1 below).
DI void accumulate_recs(const K3Args& a3, const K4Args& a, int s, int h, float4& pacc, float& mrun) {
  const long off = a.acc_off + static_cast<long>(s) * a.H + h;
  float4 v[8];
  float mr[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    if (r < a3.world) {
      v[r] = __ldcg(reinterpret_cast<const float4*>(a3.rb[r] + off));
      mr[r] = a.rec_unit ? 0.f : __ldcg(a3.rb[r] + static_cast<long>(s) * a3.rec_stride);
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {  // fixed summation order (rank order)
    if (r >= a3.world) break;
    if (mr[r] > mrun) {
      const float q = (mrun == neg_inf()) ? 0.f : __expf(mrun - mr[r]);
      pacc.x *= q;
      pacc.y *= q;
      pacc.z *= q;
      pacc.w *= q;
      mrun = mr[r];
    }
    const float sc = __expf(mr[r] - mrun);
    pacc.x = fmaf(v[r].x, sc, pacc.x);
    pacc.y = fmaf(v[r].y, sc, pacc.y);
    pacc.z = fmaf(v[r].z, sc, pacc.z);
    pacc.w = fmaf(v[r].w, sc, pacc.w);
  }
}

DI void smooth_block(const K3Args& a3, const K4Args& a, int blk, unsigned long long* tr) {
  __shared__ float s_m[8], s_w[8];
  __shared__ float s_cw[8][32];  // credit-fused smoothing: per-slot weights w_k and ids
  __shared__ int s_cid[8][32];
  __shared__ float4 red[kSmGroups][kSmCols];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cl = threadIdx.x % kSmCols, grp = threadIdx.x / kSmCols;
  const long e0 = static_cast<long>(blk) * kSmCols * 4;
  const long total = static_cast<long>(a.M) * a.H;
  const int s0 = static_cast<int>(e0 / a.H);
  const int s1 = static_cast<int>((min(e0 + kSmCols * 4, total) - 1) / a.H);
  const long e = e0 + static_cast<long>(cl) * 4;
  const bool in = e < total;
  const int s = in ? static_cast<int>(e / a.H) : s0;
  const int h = in ? static_cast<int>(e - static_cast<long>(s) * a.H) : 0;
  const bool active = in && a.mask_start[s] != 0;
  // The row warps merge their row's statistics first (their loads go out ahead
  // of the partial stream); every warp then streams its strided subset of the
  // partials, 8 loads in flight, with an online rescale to the running max
  // (pacc = sum_p e^{m_p - mrun} acc_p, fixed order), so the statistics are
  // needed only for the final scale and both latencies overlap.
#ifdef DINFER_K34_FINE
  if (tr != nullptr) tr[0] = globaltimer_ns();  // (fine trace) smoothing body start
#endif
  if (warp <= s1 - s0) {
    float m, l;
    int vs;
    const int i = s0 + warp;
    row_stats(a3, i, lane, m, vs, l);
    float extra = 0.f;
    if (a.cids0 != nullptr && a.mask_start[i]) {
      // credit-fused smoothing (f4): this step's credit update recomputed from
      // the step-start snapshot with the selection's own helpers, then
      // p~ = softmax(f~) = (e^{f-m} + w_v [v credited]) / (l + sum w)
      const bool slot = lane < a3.K;
      const long cb = static_cast<long>(i) * a3.K;
      int cid = slot ? a.cids0[cb + lane] : -1;
      float cv = slot ? a.cval0[cb + lane] : 0.f;
      const float fc = slot ? a3.rb[0][static_cast<long>(i) * a3.rec_stride + kStatWords + lane] : 0.f;
      credit_update_slots(a3.c_beta, a3.c_gamma, slot, vs, __frcp_rn(l), cid, cv);
      float w = 0.f;
      if (cid >= 0) {
        float ft;
        w = credit_fuse_slot(a3.c_alpha, cid, cv, vs, m, fc, ft);
      }
      s_cw[warp][lane] = w;
      s_cid[warp][lane] = cid;
      extra = warp_sum(w);
    }
    if (lane == 0) {
      s_m[warp] = m;
      s_w[warp] = a.alpha_t / (l + extra);
    }
#ifdef DINFER_K34_FINE
    if (tr != nullptr) tr[4] = globaltimer_ns();  // (fine trace) row stats merged
#endif
  }
  float4 pacc = make_float4(0.f, 0.f, 0.f, 0.f);
  float mrun = neg_inf();
  if (a.rec_mode) {
    if (active && grp == 0) accumulate_recs(a3, a, s, h, pacc, mrun);
    // K12 record mode: the step's record accumulator is zeroed for the next
    // step once read (same thread: the stores follow the loads of the same
    // addresses; a double-buffered record zeroes the other slot)
    if (a.zero_acc != nullptr && in && grp == 0)
      *reinterpret_cast<float4*>(a.zero_acc + static_cast<long>(s) * a.H + h) = make_float4(0.f, 0.f, 0.f, 0.f);
  } else if (active) {
    accumulate_parts<kSmBatchH, true>(a, s, h, grp, pacc, mrun);  // fp16 per-group partials
  }
  __syncthreads();
  if (tr != nullptr) tr[2] = globaltimer_ns();
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (active && mrun != neg_inf()) {
    const float sc = a.rec_unit ? 1.f : __expf(mrun - s_m[s - s0]);
    acc = make_float4(pacc.x * sc, pacc.y * sc, pacc.z * sc, pacc.w * sc);
  }
  red[grp][cl] = acc;
  __syncthreads();
  if (grp == 0 && active) {
    for (int g = 1; g < kSmGroups; ++g) {
      const float4 r = red[g][cl];
      acc.x += r.x;
      acc.y += r.y;
      acc.z += r.z;
      acc.w += r.w;
    }
    if (a.cids0 != nullptr) {  // + sum_k w_k E[id_k, h..h+3] over the row's credited tokens
      const int rr = s - s0;
      for (int k = 0; k < a3.K; ++k) {
        const int id = s_cid[rr][k];
        if (id < 0 || id >= a3.V_total) continue;  // invalid ids are flagged by the selection
        const float wk = s_cw[rr][k];
        const uint2 ev = *reinterpret_cast<const uint2*>(a.E + static_cast<long>(id) * a.H + h);
        const __nv_bfloat162 e01 = *reinterpret_cast<const __nv_bfloat162*>(&ev.x);
        const __nv_bfloat162 e23 = *reinterpret_cast<const __nv_bfloat162*>(&ev.y);
        acc.x = fmaf(wk, __low2float(e01), acc.x);
        acc.y = fmaf(wk, __high2float(e01), acc.y);
        acc.z = fmaf(wk, __low2float(e23), acc.z);
        acc.w = fmaf(wk, __high2float(e23), acc.w);
      }
    }
    const float w = s_w[s - s0];
    const uint2 em = *reinterpret_cast<const uint2*>(a.e_mask + h);
    const __nv_bfloat162 e01 = *reinterpret_cast<const __nv_bfloat162*>(&em.x);
    const __nv_bfloat162 e23 = *reinterpret_cast<const __nv_bfloat162*>(&em.y);
    float4 o;
    o.x = fmaf(w, acc.x, __low2float(e01));
    o.y = fmaf(w, acc.y, __high2float(e01));
    o.z = fmaf(w, acc.z, __low2float(e23));
    o.w = fmaf(w, acc.w, __high2float(e23));
    *reinterpret_cast<float4*>(a.out + e) = o;
    if (a.emb != nullptr) {  // next-iteration input of a (possibly) still-masked row: bf16(e_{t+1})
      const __nv_bfloat162 o01 = __floats2bfloat162_rn(o.x, o.y), o23 = __floats2bfloat162_rn(o.z, o.w);
      uint2 ob;
      ob.x = *reinterpret_cast<const uint32_t*>(&o01);
      ob.y = *reinterpret_cast<const uint32_t*>(&o23);
      *reinterpret_cast<uint2*>(a.emb + e) = ob;
    }
  } else if (grp == 0 && in && a.emb != nullptr) {  // decided at step start: its token's embedding row
    const long tok = a.tokens[s];
    *reinterpret_cast<uint2*>(a.emb + e) = *reinterpret_cast<const uint2*>(a.E + tok * a.H + h);
  }
  if (a.emb != nullptr) {  // count this block's rows as written (the selection block waits for them)
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      for (int r = s0; r <= s1; ++r) atomicAdd(a.rowdone + r, 1);
    }
  }
}

// K3+K4 in one launch: blocks [0, B) select/commit batch rows, blocks >= B
// (only with smoothing) write the smoothed embeddings.  Both read only what
// K1 / K2 / the allgather produced (plus the step-start mask snapshot).
__global__ void __launch_bounds__(kK3Threads, 1) k34_select_smooth(const __grid_constant__ K3Args a3in, const __grid_constant__ K4Args a4in) {
  unsigned long long* tr =
      (a3in.trace != nullptr && threadIdx.x == 0 && blockIdx.x < kTraceK34) ? a3in.trace + blockIdx.x * 5 : nullptr;
  if (tr != nullptr) {
    tr[0] = globaltimer_ns();
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    tr[4] = sm;
  }
  grid_dep_wait();  // K1 / K2 / allgather results visible
  if (tr != nullptr) tr[1] = globaltimer_ns();
  grid_dep_launch_dependents();
  K3Args a3 = a3in;
  K4Args a4 = a4in;
  unsigned epoch = 0;
  __shared__ const float* s_rb[32];  // record base of rank r (read in place; K1b: vocab group r)
  if (a3.xflags != nullptr) {
    // peer-memory exchange: rank r's record of this epoch is complete in slot
    // (epoch & 1) of its exchange buffer once r's flag here reads epoch + 1
    epoch = *reinterpret_cast<volatile unsigned*>(a3.xctl);
    const unsigned par = epoch & 1u;
    if (static_cast<int>(threadIdx.x) < a3.world) {
      const unsigned* f = a3.xflags + par * a3.world + threadIdx.x;
      uint32_t spins = 0;
      for (;;) {
        unsigned v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (v == epoch + 1u) break;
        __nanosleep(64);
        if (++spins > (1u << 26)) __trap();
      }
    }
    __syncthreads();
    if (a4.zero_par > 0) a4.zero_acc += (par ^ 1u) * a4.zero_par;  // the slot the NEXT step's K12 fills
  }
  if (threadIdx.x < 32) {
    const int r = threadIdx.x;
    s_rb[r] = (r >= a3.world) ? nullptr
              : (a3.rpar > 0) ? a3in.rpv[r] + (epoch & 1u) * a3.rpar
                                     : (a3.recs != nullptr ? a3.recs + r * a3.rec_words : nullptr);
  }
  __syncthreads();
  a3.rb = s_rb;
  if (a3.pdev != nullptr) {  // per-step numeric parameters from device memory (graph replay)
    a3.tau = a3.pdev[0];
    a3.theta_hi = a3.pdev[1];
    a3.theta_lo = a3.pdev[2];
    a3.c_alpha = a3.pdev[3];
    a3.c_beta = a3.pdev[4];
    a3.c_gamma = a3.pdev[5];
    a4.alpha_t = a3.pdev[6];
  }
  const int nsel = a3.B * sel_ctas_per_row(a3.S);
  if (static_cast<int>(blockIdx.x) < nsel) {
    select_block(a3, blockIdx.x, tr);
  } else {
    smooth_block(a3, a4, blockIdx.x - nsel, tr);
  }
  if (tr != nullptr) tr[3] = globaltimer_ns();
  if (a3.xflags != nullptr) {  // the last block advances the exchange epoch
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(a3.xctl + 2, 1u) == gridDim.x - 1) {
        a3.xctl[2] = 0u;
        a3.xctl[0] = epoch + 1u;
      }
    }
  }
}

}  // namespace

cudaError_t launch_k34(const K3Args& a3, const K4Args* a4, cudaStream_t st, bool pdl) {
  {  // same smem carveout as K1/K2 (no L1/smem reconfiguration between kernels)
    const cudaError_t e = ensure_func_smem(reinterpret_cast<const void*>(k34_select_smooth), 0, 100);
    if (e != cudaSuccess) return e;
  }
  int nsm = 0;
  K4Args f{};
  if (a4 != nullptr) {
    f = *a4;
    nsm = static_cast<int>((static_cast<long>(f.M) * f.H / 4 + kSmCols - 1) / kSmCols);
  }
  return launch_ex(k34_select_smooth, dim3(a3.B * ((a3.S + kSelPos - 1) / kSelPos) + nsm), dim3(kK3Threads), 0, st,
                   pdl, a3, f);
}

}  // namespace dinfer
