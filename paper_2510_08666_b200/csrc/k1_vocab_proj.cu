// K1 vocab_proj -- LM-head contraction fused with the softmax-statistics
// epilogue (PAPER.md:95-96 logits; P:278 softmax; P:305 v* = argmax).
//
//   logits^T[v, s] = W[v, :] . h[s, :]       (swap-AB: vocab on UMMA M = 128,
//                                              positions on UMMA N = M_pos)
// Per (position s) the kernel produces m = max_v f, v* = lowest argmax id,
// l = sum_v exp(f - m) over this rank's vocab shard; the logits never leave
// TMEM except (a) the raw value of credited tokens (credit fuse)
// and (b) -- only when smoothing is on -- an fp32 copy for the smoothing mix
// (DESIGN.md "K2 v1").
//
// Structure (one CTA per SM, persistent over a contiguous vocab slab):
//   warp 4    TMA producer: W chunks [128 rows x 64 k] (SWIZZLE_128B) into a
//             `stages`-deep ring; hidden either resident (loaded once) or
//             streamed with each W chunk.
//   warp 5    MMA issuer: tcgen05.mma.cta_group::1.kind::f16 128xNx16, fp32
//             accumulator double-buffered in TMEM (2 x N columns).
//   warps 0-3 epilogue: tcgen05.ld 32 columns per lane (lane = vocab row),
//             warp-shuffle reduce-scatter of (m, idx, l) across the 32 rows
//             (31 pairwise merges per 32x32 block), running merge per column.
//   End: cross-warp merge -> per-CTA partial (m, idx, l) per position, and a
//   release-ordered increment of the slab's vocab-group counter (K2 waits on
//   it).  Partials are merged downstream in a fixed order (deterministic).
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace dinfer {
namespace {

constexpr int kEpiWarps = 4;
constexpr int kThreads = (kEpiWarps + 2) * kWarpThreads;
// A pipeline stage carries two adjacent K-chunks of W (2 x [128 rows x 64 k]
// = 32 KB, 256 contiguous bytes per row): single 16 KB boxes cap TMA
// streaming at ~4.7 TB/s on B200, adjacent pairs reach ~5.6 TB/s
// (tools/hbm_stream.cu, profiles/).
constexpr int kChunksPerStage = 2;
// W tiles of up to kTileMax rows (N <= 128; 128 rows for larger N, whose
// double-buffered accumulators already fill the TMEM): rows [0, 128) are one
// UMMA, rows [128, 160) a second one over the next 128 rows of the chunk
// space (rows past the tile are stale and ignored).  A slab is cut into
// 32-row units (the last one may be shorter) grouped into near-equal tiles
// of <= 5 units, so tiles are loaded as one 128-row box plus 32-row boxes
// (8-row boxes only for the slab's last < 32 rows) -- short tail tiles of
// 8-row boxes streamed at a fraction of the rate (K12 trace).
constexpr int kTileMax = 160;
constexpr uint32_t kChunkBytes = kTileMax * 128;                  // chunk space: 20 KB
constexpr uint32_t kWStageBytes = kChunksPerStage * kChunkBytes;  // 40 KB
constexpr int kMaxGroups = 8;                       // N <= 256
constexpr int kUnit = 32;                           // rows per tile unit

DI int unit_row(int r0, int r1, int nu, int u) { return min(r1, r0 + u * kUnit); }
// first unit of tile t of nt tiles over nu units
DI int tile_u(int nu, int nt, int t) { return static_cast<int>(static_cast<long>(t) * nu / nt); }

__host__ __device__ inline uint32_t tmem_cols_pow2(uint32_t n) {
  uint32_t c = 32;
  while (c < n) c <<= 1;
  return c;
}

DI float pick32(const float (&x)[32], int j) {
  float r = 0.f;
#pragma unroll
  for (int q = 0; q < 32; ++q) r = (q == j) ? x[q] : r;
  return r;
}

// One reduce-scatter level: 2*O values per lane -> O values, merging with the
// partner lane (lane ^ O).  Lanes with bit O set keep the upper half.
template <int O>
DI void rs_level(float* m, int* ix, float* l, bool up) {
#pragma unroll
  for (int k = 0; k < O; ++k) {
    float km = up ? m[k + O] : m[k];
    int ki = up ? ix[k + O] : ix[k];
    float kl = up ? l[k + O] : l[k];
    const float sm = up ? m[k] : m[k + O];
    const int si = up ? ix[k] : ix[k + O];
    const float sl = up ? l[k] : l[k + O];
    const float rm = __shfl_xor_sync(0xffffffffu, sm, O);
    const int ri = __shfl_xor_sync(0xffffffffu, si, O);
    const float rl = __shfl_xor_sync(0xffffffffu, sl, O);
    stat_combine(km, ki, kl, rm, ri, rl);
    m[k] = km;
    ix[k] = ki;
    l[k] = kl;
  }
}

DI void named_bar_epi() { asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * kWarpThreads) : "memory"); }

struct Layout {
  uint32_t h_off, w_off, bar_off, misc_off, head_off, ent_off, red_off, total;
};

__host__ __device__ inline Layout make_layout(int N, int H, int stages, int h_resident, int slab_rows_max) {
  Layout L;
  const uint32_t hchunk = static_cast<uint32_t>(N) * 128u;
  const uint32_t h_slots =
      h_resident ? static_cast<uint32_t>(H / kKChunk) : static_cast<uint32_t>(stages * kChunksPerStage);
  L.h_off = 0;
  L.w_off = L.h_off + h_slots * hchunk;
  L.bar_off = L.w_off + static_cast<uint32_t>(stages) * kWStageBytes;
  L.misc_off = L.bar_off + static_cast<uint32_t>(2 * stages + 5) * 8u;
  L.head_off = L.misc_off + 16u;
  L.ent_off = L.head_off + static_cast<uint32_t>(slab_rows_max) * 4u;
  L.red_off = (L.ent_off + 3u * kMaxCreditEnt * 2u + 15u) & ~15u;
  L.total = L.red_off + static_cast<uint32_t>(kEpiWarps * N * 3) * 4u;
  return L;
}

__global__ void __launch_bounds__(kThreads, 1)
    k1_vocab_proj(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_w8,
                  const __grid_constant__ CUtensorMap map_w32, const __grid_constant__ CUtensorMap map_h,
                  const K1Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const Layout L = make_layout(a.N, a.H, a.stages, a.h_resident, a.slab_rows_max);
  const int warp = threadIdx.x / kWarpThreads;
  const int lane = threadIdx.x % kWarpThreads;
  const int N = a.N;
  const uint32_t hchunk = static_cast<uint32_t>(N) * 128u;

  uint8_t* h_sm = smem + L.h_off;
  uint8_t* w_sm = smem + L.w_off;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty = full + a.stages;
  uint64_t* tfull = empty + a.stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + L.misc_off);  // tmem base, last flag, entry count
  int* head = reinterpret_cast<int*>(smem + L.head_off);
  int16_t* ent_s = reinterpret_cast<int16_t*>(smem + L.ent_off);
  int16_t* ent_k = ent_s + kMaxCreditEnt;
  int16_t* ent_next = ent_k + kMaxCreditEnt;
  float* red = reinterpret_cast<float*>(smem + L.red_off);

  // Contiguous slab of vocab rows [r0, r1): the vocabulary is cut into VG
  // groups on 64-row chunk boundaries (K2's vocab groups) and each group into
  // SPG slabs balanced at 8-row granularity; slab = blockIdx.x.
  const int grp = blockIdx.x / a.SPG, q = blockIdx.x - grp * a.SPG;
  const int rg0 = a.chunk_rows * static_cast<int>(static_cast<long>(grp) * a.nchunks / a.VG);
  const int rg1 = min(a.V_local, a.chunk_rows * static_cast<int>(static_cast<long>(grp + 1) * a.nchunks / a.VG));
  const int n8 = (rg1 - rg0) / kRowGran;
  int r0 = rg0 + kRowGran * static_cast<int>(static_cast<long>(q) * n8 / a.SPG);
  int r1 = rg0 + kRowGran * static_cast<int>(static_cast<long>(q + 1) * n8 / a.SPG);
  if (a.slab_start != nullptr) {  // calibrated slabs (dinfer_balance, stats-only contexts)
    r0 = a.slab_start[blockIdx.x];
    r1 = min(a.V_local, a.slab_start[blockIdx.x + 1]);
  }
  unsigned long long t_start = 0ull;  // calibration stamp: from the dependency wait (thread 0)
  const bool big = 4 * N <= 512;                        // tiles of up to 160 rows (two UMMA outputs)
  const int umax = big ? kTileMax / kUnit : kTileRows / kUnit;
  const int nu = (r1 - r0 + kUnit - 1) / kUnit;          // units (the last may be short)
  const int ntiles = (nu + umax - 1) / umax;
  const uint32_t tmem_cols = tmem_cols_pow2((big ? 4u : 2u) * N);
  const uint32_t acc_stride = (big ? 2u : 1u) * N;       // TMEM columns per accumulator buffer

  if (a.trace != nullptr && threadIdx.x == 0) { a.trace[blockIdx.x * 5 + 0] = globaltimer_ns(); uint32_t sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm)); a.trace[blockIdx.x * 5 + 4] = sm; }
  if (warp == 4 && lane == 0) {
    prefetch_tmap(&map_w);
    prefetch_tmap(&map_w8);
    prefetch_tmap(&map_w32);
    prefetch_tmap(&map_h);
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps * kWarpThreads);
    }
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(&misc[0], tmem_cols);
  if (warp < kEpiWarps) {
    for (int r = threadIdx.x; r < r1 - r0; r += kEpiWarps * kWarpThreads) head[r] = -1;
    if (threadIdx.x == 0) misc[2] = 0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = misc[0];
  // The next kernel (K2 / K3) may be scheduled onto SMs as they free up.
  grid_dep_launch_dependents();

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      grid_dep_wait();  // hidden may be produced by the preceding kernel
      const uint64_t pol_w = policy_evict_first();  // W is streamed exactly once
      const uint64_t pol_h = policy_evict_last();   // hidden is re-read by every CTA
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int row0 = unit_row(r0, r1, nu, tile_u(nu, ntiles, t));
        const int rows = unit_row(r0, r1, nu, tile_u(nu, ntiles, t + 1)) - row0;
        for (int kc0 = 0; kc0 < a.num_kc; kc0 += kChunksPerStage) {
          mbar_wait(&empty[stage], phase ^ 1u);
          // hidden chunk kc rides with W chunk kc: every stage when streamed,
          // only tile 0 when resident (it then stays in slot kc).
          const bool with_h = !a.h_resident || t == 0;
          const uint32_t bytes =
              kChunksPerStage * (static_cast<uint32_t>(rows) * 128u + (with_h ? hchunk : 0u));
          mbar_expect_tx(&full[stage], bytes);
#pragma unroll
          for (int j = 0; j < kChunksPerStage; ++j) {
            const int kc = kc0 + j;
            uint8_t* dst = w_sm + stage * kWStageBytes + j * kChunkBytes;
            // row r lands at dst + r * 128 (SW128 atoms of 8 rows): one 128-row
            // box, 32-row boxes, 8-row boxes for the slab's last < 32 rows
            int r = 0;
            if (rows >= kTileRows) {
              tma_load_2d(dst, &map_w, &full[stage], kc * kKChunk, row0, pol_w);
              r = kTileRows;
            }
            for (; r + kUnit <= rows; r += kUnit)
              tma_load_2d(dst + r * 128, &map_w32, &full[stage], kc * kKChunk, row0 + r, pol_w);
            for (; r < rows; r += kRowGran)
              tma_load_2d(dst + r * 128, &map_w8, &full[stage], kc * kKChunk, row0 + r, pol_w);
            if (with_h)
              tma_load_2d(h_sm + (a.h_resident ? kc : stage * kChunksPerStage + j) * hchunk, &map_h, &full[stage],
                          kc * kKChunk, 0, pol_h);
          }
          if (++stage == a.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    // warp-collective issue with per-stage descriptors advanced by constant
    // offsets (common.cuh mma_bf16_warp: no per-MMA ELECT waterfall)
    const uint32_t idesc = idesc_bf16(kTileRows, N, false, false);
    int stage = 0;
    uint32_t phase = 0;
    for (int t = 0; t < ntiles; ++t) {
      const int buf = t & 1;
      const uint32_t use = static_cast<uint32_t>(t >> 1);
      const bool two = unit_row(r0, r1, nu, tile_u(nu, ntiles, t + 1)) - unit_row(r0, r1, nu, tile_u(nu, ntiles, t)) >
                       kTileRows;
      mbar_wait(&tempty[buf], (use & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t d = tmem_base + static_cast<uint32_t>(buf) * acc_stride;
      for (int kc0 = 0; kc0 < a.num_kc; kc0 += kChunksPerStage) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0 && a.trace != nullptr && t == 0 && kc0 == 0) a.trace[blockIdx.x * 5 + 1] = globaltimer_ns();
        const uint64_t a0 = sdesc_sw128(smem_u32(w_sm + stage * kWStageBytes), 16, 1024);
        const uint64_t b0 = sdesc_sw128(smem_u32(h_sm + (a.h_resident ? kc0 : stage * kChunksPerStage) * hchunk), 16,
                                        1024);
#pragma unroll
        for (int j = 0; j < kChunksPerStage; ++j)
#pragma unroll
          for (int k = 0; k < kKChunk / 16; ++k) {
            const uint64_t bd = sdesc_add(b0, j * hchunk + k * 32);
            const uint32_t acc = ((kc0 + j) | k) != 0;
            mma_bf16_warp(d, sdesc_add(a0, j * kChunkBytes + k * 32), bd, idesc, acc);
            if (two) mma_bf16_warp(d + N, sdesc_add(a0, j * kChunkBytes + kTileRows * 128 + k * 32), bd, idesc, acc);
          }
        mma_commit_warp(&empty[stage]);  // frees the smem slot when these MMAs finish
        if (++stage == a.stages) {
          stage = 0;
          phase ^= 1u;
        }
      }
      mma_commit_warp(&tfull[buf]);  // accumulator ready for the epilogue
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    // Credited (position, slot) entries whose token lives in this slab: their
    // raw logits are captured for the credit fuse.  Rows decided at step start
    // are frozen (reading c7) and skipped.  Runs while the first W chunks fly.
    grid_dep_wait();  // mask / credit ids of the previous step's commit visible
    if (a.wdur != nullptr && threadIdx.x == 0) t_start = globaltimer_ns();
    // record stats rows of this step (slot (epoch & 1) of a double-buffered record)
    float* recw = a.rec;
    if (a.rec_par > 0) recw += (*reinterpret_cast<const volatile unsigned*>(a.rec_ctl) & 1u) * a.rec_par;
    if (a.mask_snap != nullptr && blockIdx.x == 0)
      for (int s = threadIdx.x; s < a.M; s += kEpiWarps * kWarpThreads) a.mask_snap[s] = a.block_start ? 1 : a.mask[s];
    if (a.cids_snap != nullptr && blockIdx.x == 0)
      for (int e = threadIdx.x; e < a.M * a.K; e += kEpiWarps * kWarpThreads) {
        a.cids_snap[e] = a.block_start ? -1 : a.credit_ids[e];
        a.cval_snap[e] = a.block_start ? 0.f : a.credit_val[e];
      }
    if (a.credit_ids != nullptr && !a.block_start) {  // block start: no credited token yet
      const int stride = kStatWords + a.K;
      for (int e = threadIdx.x; e < a.M * a.K; e += kEpiWarps * kWarpThreads) {
        const int s = e / a.K, k = e - s * a.K;
        if (!a.mask[s]) continue;
        const int id = a.credit_ids[e];
        if (id < 0) continue;
        const int lv = id - a.v_offset;
        if (lv < 0 || lv >= a.V_local) {  // owned by another rank
          if (blockIdx.x == 0) recw[s * stride + kStatWords + k] = neg_inf();
          continue;
        }
        if (lv < r0 || lv >= r1) continue;
        const int slot = static_cast<int>(atomicAdd(&misc[2], 1u));
        if (slot >= kMaxCreditEnt) {
          atomicOr(a.err, kErrCreditEntOverflow);
          continue;
        }
        ent_s[slot] = static_cast<int16_t>(s);
        ent_k[slot] = static_cast<int16_t>(k);
        ent_next[slot] = static_cast<int16_t>(atomicExch(&head[lv - r0], slot));
      }
    }
    named_bar_epi();
    const int ng = N / 32;
    float Rm[kMaxGroups];
    int Ri[kMaxGroups];
    float Rl[kMaxGroups];
#pragma unroll
    for (int g = 0; g < kMaxGroups; ++g) {
      Rm[g] = neg_inf();
      Ri[g] = INT_MAX;
      Rl[g] = 0.f;
    }
    const bool up16 = lane & 16, up8 = lane & 8, up4 = lane & 4, up2 = lane & 2, up1 = lane & 1;
    const int stride = kStatWords + a.K;
    for (int t = 0; t < ntiles; ++t) {
      const int buf = t & 1;
      const uint32_t use = static_cast<uint32_t>(t >> 1);
      mbar_wait(&tfull[buf], use & 1u);
      tc_fence_after();
      const int trow0 = unit_row(r0, r1, nu, tile_u(nu, ntiles, t));
      const int trows = unit_row(r0, r1, nu, tile_u(nu, ntiles, t + 1)) - trow0;
      for (int u = 0; u * kTileRows < trows; ++u) {  // the tile's UMMA outputs: rows [128 u, 128 u + 128)
      const int row0 = trow0 + u * kTileRows;
      const int rows = min(kTileRows, trows - u * kTileRows);
      const int rit = warp * 32 + lane;
      const bool valid = rit < rows;
      const int lv = row0 + rit;
      const int gid = a.v_offset + lv;
      const int ent0 = valid ? head[lv - r0] : -1;
#pragma unroll
      for (int g = 0; g < kMaxGroups; ++g) {
        if (g < ng) {
          float x[32];
          tmem_ld32(tmem_base + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(buf) * acc_stride +
                        static_cast<uint32_t>(u * N + g * 32),
                    x);
          if (a.flog != nullptr && valid) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = g * 32 + j;
              if (col < a.M) a.flog[static_cast<long>(col) * a.V_local + lv] = x[j];
            }
          }
          for (int e = ent0; e >= 0; e = ent_next[e]) {
            const int s = ent_s[e] - g * 32;
            if (s >= 0 && s < 32) recw[(g * 32 + s) * stride + kStatWords + ent_k[e]] = pick32(x, s);
          }
          float m[32], l[32];
          int ix[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            m[j] = valid ? x[j] : neg_inf();
            ix[j] = valid ? gid : INT_MAX;
            l[j] = valid ? 1.f : 0.f;
          }
          rs_level<16>(m, ix, l, up16);
          rs_level<8>(m, ix, l, up8);
          rs_level<4>(m, ix, l, up4);
          rs_level<2>(m, ix, l, up2);
          rs_level<1>(m, ix, l, up1);
          stat_combine(Rm[g], Ri[g], Rl[g], m[0], ix[0], l[0]);  // lane = column g*32+lane
        }
      }
      }  // u
      tc_fence_before();
      mbar_arrive(&tempty[buf]);
    }
    if (a.trace != nullptr && threadIdx.x == 0) a.trace[blockIdx.x * 5 + 2] = globaltimer_ns();
    if (a.wdur != nullptr && threadIdx.x == 0) a.wdur[blockIdx.x] = static_cast<unsigned>(globaltimer_ns() - t_start);
    // cross-warp merge (fixed warp order)
#pragma unroll
    for (int g = 0; g < kMaxGroups; ++g) {
      if (g < ng) {
        float* r = red + (warp * N + g * 32 + lane) * 3;
        r[0] = Rm[g];
        r[1] = __int_as_float(Ri[g]);
        r[2] = Rl[g];
      }
    }
    named_bar_epi();
    for (int col = threadIdx.x; col < a.M; col += kEpiWarps * kWarpThreads) {
      float m = red[col * 3 + 0], l = red[col * 3 + 2];
      int ix = __float_as_int(red[col * 3 + 1]);
      for (int w = 1; w < kEpiWarps; ++w) {
        const float* r = red + (w * N + col) * 3;
        stat_combine(m, ix, l, r[0], __float_as_int(r[1]), r[2]);
      }
      // partials are column-major [M][grid] so a column range is contiguous
      reinterpret_cast<float4*>(a.part)[static_cast<long>(col) * gridDim.x + blockIdx.x] =
          make_float4(m, __int_as_float(ix), l, 0.f);
    }
    // Publish: this slab's logits (flog), captured credited logits and
    // partial statistics are complete -> count it towards its vocab group, so
    // K2's CTAs for that group can start without waiting for the whole grid.
    // The per-CTA partials are merged downstream (K2 needs only the group
    // max, K3 merges all slabs in a fixed order), off K1's critical path.
    __threadfence();
    named_bar_epi();
    if (threadIdx.x == 0 && a.grp_cnt != nullptr) {
      __threadfence();
      atomicAdd(&a.grp_cnt[grp], 1u);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc(tmem_base, tmem_cols);
  if (a.trace != nullptr && threadIdx.x == 0) a.trace[blockIdx.x * 5 + 3] = globaltimer_ns();
}

}  // namespace

size_t k1_smem_bytes(int N, int H, int stages, int h_resident, int slab_rows_max) {
  return make_layout(N, H, stages, h_resident, slab_rows_max).total + 1024;
}

cudaError_t launch_k1(const CUtensorMap& map_w, const CUtensorMap& map_w8, const CUtensorMap& map_w32,
                      const CUtensorMap& map_h, const K1Args& a, int grid, size_t smem, cudaStream_t st, bool pdl) {
  {
    const cudaError_t e = ensure_func_smem(reinterpret_cast<const void*>(k1_vocab_proj), smem);
    if (e != cudaSuccess) return e;
  }
  return launch_ex(k1_vocab_proj, dim3(grid), dim3(kThreads), smem, st, pdl, map_w, map_w8, map_w32, map_h, a);
}

}  // namespace dinfer
