// K3 select_commit -- combine the per-rank statistics, credit update + fuse,
// threshold / hierarchical selection, commit.  K4 smooth_finalize -- the
// iteration-smoothing output e_{t+1} for positions still masked.
//
// K3: one CTA per batch row, one thread per position (S <= 1024).
//   combine   m = max_r m_r, v* = v*_r of the maximiser (lowest id on ties),
//             l = sum_r l_r e^{m_r - m}; lse = m + ln l; p* = 1/l
//   credit    undecided rows: C <- beta*C; C[v*] += p*^gamma  (Eq. credit-update,
//             P:306-313) on K sparse slots (exactly the dense table: untouched
//             tokens have C = 0); fuse f~ = f + alpha ln(1+C) (Eq. logits-fuse,
//             P:317-322); only credited tokens change, so
//             lse~ = m + ln(l + sum_{cred} e^{f_v - m}((1+C_v)^alpha - 1)),
//             v~ = argmax_{cred u {v*}} f~, p~ = e^{f~_{v~} - lse~}.
//   select    threshold (strict '>', fallback max) or hierarchical
//             (maximal runs of undecided positions; per run the
//             best position, ties nearest the run centre then lower index,
//             if p~ > theta_lo), via ballots and shared-memory atomics.
//   commit    tokens[s] = v~, mask[s] = 0, committed[s] = 1
// K4: e_{t+1}[s,:] = e_mask + alpha_t * (sum_p acc_p[s,:] e^{m_p - m}) / l
//     for rows still undecided (App. A.1).
#include <climits>

#include "common.cuh"
#include "kernels.h"

#include <cuda_bf16.h>

namespace dinfer {
namespace {

constexpr int kMaxS = 1024;

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

__global__ void k3_select_commit(const K3Args a) {
  __shared__ uint32_t s_und[kMaxS / 32];
  __shared__ uint32_t s_reg[kMaxS / 32];
  __shared__ int s_runA[kMaxS];
  __shared__ unsigned long long s_runkey[kMaxS];
  __shared__ unsigned long long s_best;

  const int b = blockIdx.x;
  const int s = threadIdx.x;
  const int nwords = blockDim.x / 32;
  const bool valid = s < a.S;
  const int i = b * a.S + s;
  const int lane = s & 31, warp = s >> 5;
  const float thr_primary = (a.decoder == 0) ? a.tau : a.theta_hi;

  bool und = false;
  float pt = 0.f;
  int vt = 0;
  if (valid) {
    und = a.mask[i] != 0;
    // ---- combine the `world` records (fixed rank order)
    const float* r0 = a.recs + static_cast<long>(i) * a.rec_stride;
    float m = r0[0], l = r0[2];
    int vstar = __float_as_int(r0[1]);
    for (int r = 1; r < a.world; ++r) {
      const float* rr = a.recs + r * a.rec_words + static_cast<long>(i) * a.rec_stride;
      stat_combine(m, vstar, l, rr[0], __float_as_int(rr[1]), rr[2]);
    }
    const float lse = m + logf(l);
    const float pstar = 1.0f / l;
    vt = vstar;
    pt = pstar;
    if (a.use_credit && und) {
      int32_t* ids = a.credit_ids + static_cast<long>(i) * a.K;
      float* vals = a.credit_val + static_cast<long>(i) * a.K;
      const float gain = powf(pstar, a.c_gamma);
      int hit = -1, empty = -1;
      for (int k = 0; k < a.K; ++k) {
        const int id = ids[k];
        if (id < 0) {
          if (empty < 0) empty = k;
          continue;
        }
        vals[k] = a.c_beta * vals[k];
        if (id == vstar) hit = k;
      }
      if (hit >= 0) {
        vals[hit] += gain;
      } else if (empty >= 0) {
        ids[empty] = vstar;
        vals[empty] = gain;
      } else {
        atomicOr(a.err, kErrCreditSlotsFull);
      }
      // fuse over credited tokens (v* included)
      float best = m, extra = 0.f;
      int best_id = vstar;
      for (int k = 0; k < a.K; ++k) {
        const int id = ids[k];
        if (id < 0) continue;
        float fk;
        if (id == vstar) {
          fk = m;
        } else {
          fk = a.recs[static_cast<long>(i) * a.rec_stride + kStatWords + k];
          for (int r = 1; r < a.world; ++r)
            fk = fmaxf(fk, a.recs[r * a.rec_words + static_cast<long>(i) * a.rec_stride + kStatWords + k]);
        }
        const float lc = log1pf(vals[k]);
        const float ft = fk + a.c_alpha * lc;
        extra += expf(fk - m) * expm1f(a.c_alpha * lc);
        if (ft > best || (ft == best && id < best_id)) {
          best = ft;
          best_id = id;
        }
      }
      const float lse_t = m + logf(l + extra);
      vt = best_id;
      pt = expf(best - lse_t);
    }
    if (a.stats != nullptr) {
      float* st = a.stats + static_cast<long>(i) * 4;
      st[0] = m;
      st[1] = lse;
      st[2] = pt;
      st[3] = __int_as_float(vt);
    }
    a.ml[2 * i] = m;
    a.ml[2 * i + 1] = l;
  }

  // ---- selection
  bool A = und && pt > thr_primary;
  const unsigned ub = __ballot_sync(0xffffffffu, und);
  if (lane == 0) s_und[warp] = ub;
  if (a.decoder == 1) {
    const bool region = und && !(a.runs_after_hi && A);
    const unsigned rb = __ballot_sync(0xffffffffu, region);
    if (lane == 0) s_reg[warp] = rb;
    s_runA[s] = 0;
    s_runkey[s] = 0ull;
    __syncthreads();
    int first = 0, last = 0;
    unsigned long long key = 0ull;
    if (region) {
      first = run_first(s_reg, s);
      last = run_last(s_reg, s, nwords);
      if (A) atomicOr(&s_runA[first], 1);
      const int dist = abs(2 * s - first - last);
      key = (static_cast<unsigned long long>(__float_as_uint(pt)) << 32) |
            (static_cast<unsigned long long>(0xFFFF - dist) << 16) | static_cast<unsigned long long>(0xFFFF - s);
      atomicMax(&s_runkey[first], key);
    }
    __syncthreads();
    if (region && !s_runA[first] && s_runkey[first] == key && pt > a.theta_lo) A = true;
  }
  if (s == 0) s_best = 0ull;
  const int anyA = __syncthreads_or(A);
  if (!anyA) {  // fallback: the undecided position with max p~ (lowest index on ties)
    if (und) {
      const unsigned long long key =
          (static_cast<unsigned long long>(__float_as_uint(pt)) << 32) | static_cast<unsigned long long>(0xFFFFFFFFu - s);
      atomicMax(&s_best, key);
    }
    __syncthreads();
    A = und && s_best != 0ull && static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(s_best & 0xFFFFFFFFull)) == s;
  }

  // ---- commit
  if (valid) {
    a.committed[i] = A ? 1 : 0;
    if (A) {
      a.tokens[i] = vt;
      a.mask[i] = 0;
    }
  }
}

__global__ void k4_smooth_finalize(const K4Args a) {
  const int h4 = a.H / 4;
  const long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long>(a.M) * h4) return;
  const int s = static_cast<int>(t / h4);
  const int h = static_cast<int>(t - static_cast<long>(s) * h4) * 4;
  if (!a.mask[s]) return;  // only rows still masked get e_{t+1}
  const float m = a.ml[2 * s], l = a.ml[2 * s + 1];
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int p = 0; p < a.nparts; ++p) {
    const float4 v =
        __ldcg(reinterpret_cast<const float4*>(a.acc + p * a.acc_stride + static_cast<long>(s) * a.H + h));
    const float sc = (a.m_part == nullptr) ? 1.f : __expf(a.m_part[p * a.m_stride + static_cast<long>(s) * a.m_rowstride] - m);
    acc.x = fmaf(v.x, sc, acc.x);
    acc.y = fmaf(v.y, sc, acc.y);
    acc.z = fmaf(v.z, sc, acc.z);
    acc.w = fmaf(v.w, sc, acc.w);
  }
  const float w = a.alpha_t / l;
  const uint2 em = *reinterpret_cast<const uint2*>(a.e_mask + h);
  const __nv_bfloat162 e01 = *reinterpret_cast<const __nv_bfloat162*>(&em.x);
  const __nv_bfloat162 e23 = *reinterpret_cast<const __nv_bfloat162*>(&em.y);
  float4 o;
  o.x = fmaf(w, acc.x, __low2float(e01));
  o.y = fmaf(w, acc.y, __high2float(e01));
  o.z = fmaf(w, acc.z, __low2float(e23));
  o.w = fmaf(w, acc.w, __high2float(e23));
  *reinterpret_cast<float4*>(a.out + static_cast<long>(s) * a.H + h) = o;
}

}  // namespace

cudaError_t launch_k3(const K3Args& a, cudaStream_t st) {
  const int threads = ((a.S + 31) / 32) * 32;
  k3_select_commit<<<a.B, threads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_k4(const K4Args& a, cudaStream_t st) {
  const long n = static_cast<long>(a.M) * (a.H / 4);
  const int threads = 256;
  const int blocks = static_cast<int>((n + threads - 1) / threads);
  k4_smooth_finalize<<<blocks, threads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace dinfer
