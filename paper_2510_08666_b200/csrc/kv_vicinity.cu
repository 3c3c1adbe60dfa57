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
// The three projections are plain GEMMs (cuBLAS, bf16 in, fp32 accumulate,
// bf16 out straight into the cache rows).  The attention is a hand-written
// split-key flash kernel: CTA = (head, 16-query tile, key split), 64-key
// tiles staged in shared memory as fp32, online softmax in base 2, per-split
// (m, l, O) partials merged by a second kernel in a fixed order.  At the
// steady-state region (block 32 + 2 x 16 looks = 64 queries) the layer is
// bound by the weight (3 H^2 bf16) and cache (2 L H bf16) reads; the
// attention's 64 x L x H x 4 flop run on CUDA cores.
#include <cublas_v2.h>
#include <cuda_bf16.h>

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

// out[lo + r][head*128 + c] = sum_s O_s 2^{m_s - m} / sum_s l_s 2^{m_s - m}
// (splits merged in index order: deterministic).
__global__ void kv_attention_merge(const AttnArgs a) {
  const long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<long>(a.R) * a.H) return;
  const int r = static_cast<int>(e / a.H), col = static_cast<int>(e - static_cast<long>(r) * a.H);
  const int head = col / kD, nheads = a.H / kD;
  float m = neg_inf();
  for (int s = 0; s < a.nsplit; ++s) m = fmaxf(m, a.mpart[(static_cast<long>(s) * nheads + head) * a.R + r]);
  float num = 0.f, den = 0.f;
  for (int s = 0; s < a.nsplit; ++s) {
    const long mi = (static_cast<long>(s) * nheads + head) * a.R + r;
    const float ms = a.mpart[mi];
    if (ms == neg_inf()) continue;  // a split with no keys
    const float w = ex2(ms - m);
    num = fmaf(a.opart[(static_cast<long>(s) * a.R + r) * a.H + col], w, num);
    den = fmaf(a.lpart[mi], w, den);
  }
  a.out[static_cast<long>(a.lo + r) * a.H + col] = num / den;
}

}  // namespace
}  // namespace dinfer

using namespace dinfer;

struct dinfer_kv {
  dinfer_kv_shape shp{};
  cudaStream_t stream = nullptr;
  cublasHandle_t blas = nullptr;
  int num_sms = 0;
  uint16_t* Q = nullptr;  // [L][H]
  float* opart = nullptr;
  float* mpart = nullptr;
  float* lpart = nullptr;
  size_t part_rows = 0;   // capacity of opart in rows of H
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
  c->part_rows = static_cast<size_t>(s->L) * 4 + 256;
  const size_t nml = c->part_rows * (s->H / kD);
  bool ok = cudaMalloc(&c->Q, LH * 2) == cudaSuccess && cudaMalloc(&c->opart, c->part_rows * s->H * 4) == cudaSuccess &&
            cudaMalloc(&c->mpart, nml * 4) == cudaSuccess && cudaMalloc(&c->lpart, nml * 4) == cudaSuccess;
  if (ok) ok = cublasCreate(&c->blas) == CUBLAS_STATUS_SUCCESS;
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
  if (c->blas != nullptr) cublasDestroy(c->blas);
  cudaFree(c->Q);
  cudaFree(c->opart);
  cudaFree(c->mpart);
  cudaFree(c->lpart);
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
  // ---- K.Update + queries: Y[R, H] = X[lo:hi] W^T (bf16 out, fp32 accumulate), cuBLAS
  // column-major view: Y^T [H x R] = W^T^T ... = op_T(W as [H_in x H_out]) * X^T [H_in x R]
  if (cublasSetStream(c->blas, c->stream) != CUBLAS_STATUS_SUCCESS) return DINFER_ERR_CUDA;
  const float one = 1.f, zero = 0.f;
  const long xoff = static_cast<long>(lo) * H;
  struct Proj {
    const uint16_t* W;
    uint16_t* Y;
  } proj[3] = {{Wk, Kc + xoff}, {Wv, Vc + xoff}, {Wq, c->Q}};
  for (const Proj& pj : proj) {
    if (cublasGemmEx(c->blas, CUBLAS_OP_T, CUBLAS_OP_N, H, R, H, &one, pj.W, CUDA_R_16BF, H, X + xoff, CUDA_R_16BF,
                     H, &zero, pj.Y, CUDA_R_16BF, H, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) !=
        CUBLAS_STATUS_SUCCESS)
      return DINFER_ERR_CUDA;
  }
  // ---- attention over all L cached positions
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
  const long n = static_cast<long>(R) * H;
  kv_attention_merge<<<static_cast<unsigned>((n + 255) / 256), 256, 0, c->stream>>>(a);
  if (cudaGetLastError() != cudaSuccess) return DINFER_ERR_CUDA;
  return DINFER_OK;
}

}  // extern "C"
