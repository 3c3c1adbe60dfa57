// K12 proj_smooth -- K1 (vocab projection + softmax-statistics epilogue,
// PAPER.md:95-96) and K2 (the smoothing contraction
// acc[s,:] = sum_v exp(f[s,v] - m) E[v,:], App. A.1) fused in one
// persistent kernel, one CTA per SM, for smoothing steps with N <= 64.
//
// Why: as two kernels, K2 cannot start on an SM before K1's CTA there exits,
// and its vocab group must wait for the slowest K1 slab of the group; the
// K1 finish spread (~14 us at MoE shape) and K2's ramp-up sit on the critical
// path between two HBM streams.  Here every CTA streams its W slab and then,
// through the SAME TMA ring (no bubble: E stages are issued as soon as the
// last W stage is), the E rows of its vocab group, so HBM never idles on an
// SM while its neighbour finishes.
//
// Partition: the vocabulary is cut into VG groups of 16-row chunks; a group
// has SPG = HS slabs (one per CTA).  W phase: CTA q of group g runs the K1
// pipeline over slab q (rows at chunk granularity).  E phase: CTA q computes
// hidden slice q (HW = H / HS columns) over ALL rows of the group.  The
// softmax weights need a reference max: the CTA's OWN slab rows are processed
// first, relative to its own slab max (known the moment its W phase ends), into
// TMEM accumulator set A; the other slabs' rows follow, relative to their
// maxima (after the group counter says they are done -- by then, normally
// long ago), into set B.  The epilogue writes
//   part2[g][s][hs*HW : (hs+1)*HW] = A e^{m_own - m_g} + B e^{m_oth - m_g},
//   mref[g][s] = m_g (max over the group) -- the same partial format K2 writes,
// so K34 / the record finalize are unchanged.
//
// Shared memory: the W ring (stages x [W 32 KB + hidden]) and the E ring
// (estages x [HW h x 32 v] = 64 KB at HW = 1024, the K2 stage shape that streams
// E at ~5.7 TB/s; 16-row stages measured 4.6 TB/s) overlay the same bytes: E
// slot j is first filled only after the final consumption of every W slot it
// overlaps, so E loads start slot by slot as the W phase drains.  The logits /
// P rings alias the credit-capture tables (used only in the W phase).
//
// Warp roles (8 warps):
//   0-3  W phase: K1 epilogue (tcgen05.ld, warp-shuffle (m, idx, l) reduce-
//        scatter, credited-logit capture, raw logits -> flog); E phase: P
//        producers (P = exp(f - m_ref) as bf16 hi + lo, SWIZZLE_64B K-major
//        tiles); end: TMEM -> smem -> coalesced partial rows.
//   4    TMA producer of the shared ring: W (+ hidden) stages, then E stages.
//   5    MMA issuer: 128xNx16 bf16 UMMAs (W: swap-AB; E: A = E^T MN-major).
//   6    logits producer: flog chunks [N x 32] by TMA (own chunks after the
//        CTA's own W epilogue, others after the group counter), and m_oth.
//   7    helper: with warps 4-6, the second half of the final epilogue.
// TMEM: 512 columns.  W-phase accumulators (two UMMA outputs per tile)
// double-buffered at [0, 4N); E
// set A at [0, nsub NE), set B at [256, 256 + nsub NE), NE = 2N when the hi /
// lo P tiles are stacked into one MMA (b.stack), else N (E MMAs start only
// after the W epilogue has drained its accumulators).
#include <climits>

#include "common.cuh"
#include "kernels.h"

#include <cuda_bf16.h>

namespace dinfer {
namespace {

constexpr int kEpiWarps = 4;
constexpr int kEpiThreads = kEpiWarps * kWarpThreads;
constexpr int kThreads = (kEpiWarps + 4) * kWarpThreads;  // + TMA, MMA, logits TMA, epilogue helper
// W tiles of 1-5 units of 32 rows (the slab's 32-row chunks): rows [0, 128)
// are one UMMA (M = 128), rows [128, 160) a second one over the next 128 rows
// of the same chunk (the rows past the tile are stale and ignored).  A slab of
// n chunks is cut into ceil(n / 5) near-equal tiles, so no tile is a short
// tail: a 32-row tail tile streamed 16 stages of 8 KB through the same 4-deep
// ring, as 8-row boxes -- ~12 us for 128 KB vs ~3.3 us per 128 KB in a full
// tile (K12 trace at V/8).  Every box is 128 or 32 rows (map_w / map_w32).
constexpr int kTileMax = 160;
constexpr uint32_t kChunkSpace = kTileMax * 128;   // one K chunk of a W stage: [160 rows x 64 k] bf16 = 20 KB
constexpr uint32_t kWBytes = 2 * kChunkSpace;      // two adjacent K chunks per stage (256 B per W row)
constexpr int kMaxGroups = 2;                      // N <= 64 (32-column groups)
constexpr uint32_t kSetB = 256;                    // TMEM column of accumulator set B

struct Layout {
  uint32_t wslot, eslot, estages, ring_off, un_off, f_stage, p_stage, p_off, head_off, ent_off, bar_off, misc_off,
      m_off, red_off, total;
};

__host__ __device__ inline Layout make_layout(int N, int HW, int stages, int pstages, int slab_rows_max, int emin) {
  Layout L;
  L.wslot = (kWBytes + 2u * static_cast<uint32_t>(N) * 128u + 1023u) & ~1023u;  // W (<= 160 rows) + two hidden chunks
  L.eslot = static_cast<uint32_t>(HW) * kChunkRows12 * 2u;                        // [HW h x 32 v] bf16
  // the ring holds `stages` W slots and at least `emin` E slots (E slots past
  // the W slots' bytes start without waiting for the W phase)
  uint32_t ring = static_cast<uint32_t>(stages) * L.wslot;
  if (ring < static_cast<uint32_t>(emin) * L.eslot) ring = static_cast<uint32_t>(emin) * L.eslot;
  L.estages = ring / L.eslot;
  if (L.estages > 6u) L.estages = 6u;
  L.ring_off = 0;
  // union: logits + P rings (E phase) | credit head + entry tables (W phase)
  L.un_off = ring;
  L.f_stage = (static_cast<uint32_t>(N) * kChunkRows12 * 4u + 1023u) & ~1023u;
  L.p_stage = (2u * static_cast<uint32_t>(N) * kChunkRows12 * 2u + 1023u) & ~1023u;
  L.p_off = L.un_off + static_cast<uint32_t>(pstages) * L.f_stage;
  const uint32_t rings = static_cast<uint32_t>(pstages) * (L.f_stage + L.p_stage);
  L.head_off = L.un_off;
  L.ent_off = L.head_off + ((static_cast<uint32_t>(slab_rows_max) * 4u + 15u) & ~15u);
  const uint32_t tables = L.ent_off - L.un_off + 3u * kMaxCreditEnt * 2u;
  L.bar_off = (L.un_off + (rings > tables ? rings : tables) + 15u) & ~15u;
  // full/empty[stages], efull/eempty[estages], tfull/tempty[2], ffull/fempty/pfull/pempty[pstages], accfull, own,
  // oth, owndone
  L.misc_off = L.bar_off + (2u * stages + 2u * L.estages + 4u + 4u * pstages + 4u) * 8u;
  L.m_off = L.misc_off + 64u;  // tmem base, entry count, diagnostics words [4, 12), first-finisher flag [12]
  L.red_off = L.m_off + static_cast<uint32_t>(4 * N) * 4u;  // m_own, m_oth, scale A, scale B
  L.total = L.red_off + static_cast<uint32_t>(kEpiWarps * N * 3) * 4u;
  return L;
}

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

DI float pick32(const float (&x)[32], int j) {
  float r = 0.f;
#pragma unroll
  for (int q = 0; q < 32; ++q) r = (q == j) ? x[q] : r;
  return r;
}

DI uint32_t pack_bf16x2(float lo_elem, float hi_elem) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);
  return *reinterpret_cast<const uint32_t*>(&v);
}

DI void named_bar_epi() { asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory"); }

// Every CTA of a vocab group passes exactly once per step, after its own
// slab count and (if it has other slabs' rows to process) after seeing all
// SPG counts; the last to pass resets both counters for the next step (all
// SPG increments have happened by then).
DI void group_pass(const K2Args& b, int grp, int SPG) {
  if (atomicAdd(b.grp_pass + grp, 1u) == static_cast<unsigned>(SPG - 1)) {
    b.grp_cnt[grp] = 0u;
    b.grp_pass[grp] = 0u;
  }
}

// Diagnostics (DINFER_K12_PROBE): roles record progress in shared memory
// (plain volatile stores, no fences); a timed-out accfull wait dumps them and
// the raw mbarrier words to mapped host memory before trapping.
// Diagnostics (DINFER_K12_PROBE): roles record progress in shared memory
// (plain volatile stores, no fences); a timed-out accfull wait dumps them and
// the raw mbarrier words to mapped host memory before trapping.
#define PROBE(w, v)                  \
  do {                               \
    if (prog != nullptr) prog[w] = (v); \
  } while (0)

// First 32-row unit (chunk) of tile i of a slab of chunks [c0, c0 + n) cut into nt near-equal tiles.
DI int tile_unit(int c0, int n, int nt, int i) { return c0 + static_cast<int>(static_cast<long>(i) * n / nt); }

// The W boxes of the stage covering K chunks kc0, kc0 + 1 of the tile of
// `units` 32-row units from row0: row r of K chunk j lands at slot + j *
// kChunkSpace + r * 128 (SW128 atoms of 8 rows), so rows >= 128 start exactly
// at the second UMMA's A operand (+16 KB).  Rows past V_local are zero-filled
// by the TMA (and counted in the transaction bytes).
DI void issue_w_stage(const CUtensorMap* map_w, const CUtensorMap* map_w32, uint8_t* slot, uint64_t* bar, int row0,
                      int units, int kc0, uint64_t pol) {
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int kc = kc0 + j;
    uint8_t* dst = slot + j * kChunkSpace;
    int u = 0;
    if (units >= 4) {
      tma_load_2d(dst, map_w, bar, kc * kKChunk, row0, pol);
      u = 4;
    }
    for (; u < units; ++u) tma_load_2d(dst + u * kChunkRows12 * 128, map_w32, bar, kc * kKChunk, row0 + u * kChunkRows12, pol);
  }
}

DI void advance(int& stage, uint32_t& phase, int n) {
  if (++stage == n) {
    stage = 0;
    phase ^= 1u;
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    k12_proj_smooth(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_w32,
                    const __grid_constant__ CUtensorMap map_h, const __grid_constant__ CUtensorMap map_e,
                    const __grid_constant__ CUtensorMap map_f, const __grid_constant__ CUtensorMap map_p,
                    const K1Args a, const K2Args b) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const Layout L = make_layout(a.N, b.HW, a.stages, b.pstages, a.slab_rows_max, b.emin);
  if (L.estages < 2u) __trap();  // host geometry guarantees >= 2 E stages
  const int warp = threadIdx.x / kWarpThreads;
  const int lane = threadIdx.x % kWarpThreads;
  const int N = a.N;
  const uint32_t hchunk = static_cast<uint32_t>(N) * 128u;
  constexpr int KV = kChunkRows12;
  const uint32_t ebox = 128u * KV;                       // [64 h x 32 v] bf16 = 4 KB
  const uint32_t e_bytes = static_cast<uint32_t>(b.HW) * KV * 2u;
  const uint32_t f_bytes = static_cast<uint32_t>(N) * KV * 4u;
  const uint32_t p_half = static_cast<uint32_t>(N) * 64u;  // [N x 32] bf16, 64-B rows

  uint8_t* ring = smem + L.ring_off;
  uint8_t* f_sm = smem + L.un_off;
  uint8_t* p_sm = smem + L.p_off;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty = full + a.stages;
  uint64_t* efull = empty + a.stages;
  uint64_t* eempty = efull + L.estages;
  uint64_t* tfull = eempty + L.estages;
  uint64_t* tempty = tfull + 2;
  uint64_t* ffull = tempty + 2;
  uint64_t* fempty = ffull + b.pstages;
  uint64_t* pfull = fempty + b.pstages;
  uint64_t* pempty = pfull + b.pstages;
  uint64_t* accfull = pempty + b.pstages;
  uint64_t* own_ready = accfull + 1;    // own slab's flog / m_own complete
  uint64_t* oth_ready = own_ready + 1;  // m_oth in smem, other slabs' flog visible
  uint64_t* owndone = oth_ready + 1;    // stack mode: every own-slab E MMA complete
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + L.misc_off);  // tmem base, entry count
  volatile int* prog = b.probe != nullptr ? reinterpret_cast<volatile int*>(misc + 4) : nullptr;
  float* m_own = reinterpret_cast<float*>(smem + L.m_off);
  float* m_oth = m_own + N;
  float* scA = m_oth + N;
  float* scB = scA + N;
  int* head = reinterpret_cast<int*>(smem + L.head_off);
  int16_t* ent_s = reinterpret_cast<int16_t*>(smem + L.ent_off);
  int16_t* ent_k = ent_s + kMaxCreditEnt;
  int16_t* ent_next = ent_k + kMaxCreditEnt;
  float* red = reinterpret_cast<float*>(smem + L.red_off);

  // ---- partition: group g = chunks [gc0, gc1) of 16 rows; slab q = chunks [sc0, sc1)
  // With a calibrated partition (dinfer_balance) CTA b plays role role_of[b]
  // and the group's rows split where the two SMs' measured W rates balance.
  const int SPG = a.SPG;
  const int role = (a.role_of != nullptr) ? a.role_of[blockIdx.x] : static_cast<int>(blockIdx.x);
  const int grp = role / SPG, q = role - grp * SPG;
  const int gc0 = (a.grp_start != nullptr) ? a.grp_start[grp] : static_cast<int>(static_cast<long>(grp) * a.nchunks / a.VG);
  const int gc1 =
      (a.grp_start != nullptr) ? a.grp_start[grp + 1] : static_cast<int>(static_cast<long>(grp + 1) * a.nchunks / a.VG);
  const int nc = gc1 - gc0;
  int sc0 = gc0 + static_cast<int>(static_cast<long>(q) * nc / SPG);
  int sc1 = gc0 + static_cast<int>(static_cast<long>(q + 1) * nc / SPG);
  if (a.split != nullptr && SPG == 2) {
    const int sp = a.split[grp];
    sc0 = (q == 0) ? gc0 : sp;
    sc1 = (q == 0) ? sp : gc1;
  }
  unsigned long long t_start = 0ull;  // calibration stamps: from the dependency wait (thread 0)
  const int r0 = min(a.V_local, sc0 * KV), r1 = min(a.V_local, sc1 * KV);
  const int nunits = sc1 - sc0;                      // 32-row chunks of the slab
  const int ntiles = (nunits + 4) / 5;               // W tiles of <= 5 chunks (kTileMax rows)
  const int n_own = sc1 - sc0, n_all = nc;
  const bool has_oth = n_all > n_own;
  const int hs = q;  // hidden slice of this CTA in the E phase (SPG == HS)
  // E-phase chunk order: own slab first, then the group's other chunks in order
  auto chunk_at = [&](int j) -> int {
    if (j < n_own) return sc0 + j;
    const int o = j - n_own;
    return (o < sc0 - gc0) ? gc0 + o : sc1 + (o - (sc0 - gc0));
  };
  // trace stamps: thread 0 (start, W epilogue done, exit), the MMA thread (first W / E MMA, E MMAs done)
  const bool tr_thread = threadIdx.x == 0 || threadIdx.x == 5 * kWarpThreads;
  unsigned long long* tr = (a.trace != nullptr && tr_thread) ? a.trace + blockIdx.x * 5 : nullptr;
  unsigned long long* tr2 = (b.trace != nullptr && tr_thread) ? b.trace + blockIdx.x * 5 : nullptr;
  if (tr != nullptr && threadIdx.x == 0) {
    tr[0] = globaltimer_ns();
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    tr[4] = sm;
    if (tr2 != nullptr) tr2[4] = sm;
  }

  if (warp == 4 && lane == 0) {
    prefetch_tmap(&map_w);
    prefetch_tmap(&map_w32);
    prefetch_tmap(&map_h);
    prefetch_tmap(&map_e);
    prefetch_tmap(&map_f);
    if (b.part_tma) prefetch_tmap(&map_p);
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < static_cast<int>(L.estages); ++i) {
      mbar_init(&efull[i], 1);
      mbar_init(&eempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiThreads);
    }
    for (int i = 0; i < b.pstages; ++i) {
      mbar_init(&ffull[i], 1);
      mbar_init(&fempty[i], kEpiThreads);
      mbar_init(&pfull[i], kEpiThreads);
      mbar_init(&pempty[i], 1);
    }
    mbar_init(accfull, 1);
    mbar_init(own_ready, 1);
    mbar_init(oth_ready, 1);
    mbar_init(owndone, 1);
    fence_mbar_init();
    // W does not depend on the preceding kernel: the first ring's worth of W
    // stages is issued now (each stage's barrier expects W + hidden bytes; the
    // hidden boxes follow after grid_dep_wait)
    const int spt = a.num_kc / 2, npre = min(a.npre > 0 ? a.npre : a.stages, ntiles * spt);
    const uint64_t pol_first = (a.xbits & 4) ? policy_evict_normal() : policy_evict_first();
    const uint32_t hbytes = (a.xbits & 1) ? 0u : hchunk;
    for (int i = 0; i < npre; ++i) {
      const int t = i / spt;
      const int u0 = tile_unit(sc0, nunits, ntiles, t), nu = tile_unit(sc0, nunits, ntiles, t + 1) - u0;
      mbar_expect_tx(&full[i], 2u * (static_cast<uint32_t>(nu * KV) * 128u + hbytes));
      issue_w_stage(&map_w, &map_w32, ring + i * L.wslot, &full[i], u0 * KV, nu, (i - t * spt) * 2, pol_first);
    }
  }
  if (warp == 5) tmem_alloc(&misc[0], 512);
  if (warp < kEpiWarps) {
    for (int r = threadIdx.x; r < r1 - r0; r += kEpiThreads) head[r] = -1;
    if (threadIdx.x == 0) misc[2] = 0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = misc[0];
  grid_dep_launch_dependents();

  if (warp == 4) {
    // ------------------------------------------------------------ TMA: W (+ hidden), then E
    if (lane == 0) {
      // W and E are streamed exactly once (xbits 4 / 8: measurement variants)
      const uint64_t pol_first = (a.xbits & 4) ? policy_evict_normal() : policy_evict_first();
      const uint64_t pol_e = (a.xbits & 8) ? policy_evict_normal() : policy_evict_first();
      const uint64_t pol_h = policy_evict_last();       // hidden is re-read by every CTA
      const bool ld_h = (a.xbits & 1) == 0;
      const uint32_t hbytes = ld_h ? hchunk : 0u;
      const int spt = a.num_kc / 2, nW = ntiles * spt, npre = min(a.npre > 0 ? a.npre : a.stages, nW);
      grid_dep_wait();  // hidden may be produced by the preceding kernel
      for (int i = 0; i < npre && ld_h; ++i) {  // hidden boxes of the W stages issued before the wait
        const int kc0 = (i % spt) * 2;
        for (int j = 0; j < 2; ++j)
          tma_load_2d(ring + i * L.wslot + kWBytes + j * hchunk, &map_h, &full[i], (kc0 + j) * kKChunk, 0, pol_h);
      }
      int stage = npre % a.stages;
      uint32_t phase = (npre == a.stages) ? 1u : 0u;
      for (int idx = npre; idx < nW; ++idx) {
        const int t = idx / spt, kc0 = (idx - t * spt) * 2;
        const int u0 = tile_unit(sc0, nunits, ntiles, t), nu = tile_unit(sc0, nunits, ntiles, t + 1) - u0;
        mbar_wait(&empty[stage], phase ^ 1u);
        uint8_t* slot = ring + stage * L.wslot;
        mbar_expect_tx(&full[stage], 2u * (static_cast<uint32_t>(nu * KV) * 128u + hbytes));
        issue_w_stage(&map_w, &map_w32, slot, &full[stage], u0 * KV, nu, kc0, pol_first);
        for (int j = 0; j < 2 && ld_h; ++j)
          tma_load_2d(slot + kWBytes + j * hchunk, &map_h, &full[stage], (kc0 + j) * kKChunk, 0, pol_h);
        advance(stage, phase, a.stages);
      }
      PROBE(0, 1000 + ntiles);
      // E ring over the same bytes: slot j's first fill waits for the final
      // consumption of every W slot it overlaps (the f_i-th commit of W slot i
      // completes phase f_i - 1)
      int es = 0;
      uint32_t eph = 0;
      for (int j = 0; j < n_all; ++j) {
        const int c = chunk_at(j);
        if (j < static_cast<int>(L.estages)) {
          const int lo = static_cast<int>(static_cast<uint32_t>(j) * L.eslot / L.wslot);
          const int hi = min(a.stages - 1, static_cast<int>((static_cast<uint32_t>(j + 1) * L.eslot - 1u) / L.wslot));
          for (int i = lo; i <= hi; ++i) {
            const int fills = nW > i ? (nW - 1 - i) / a.stages + 1 : 0;
            if (fills > 0) mbar_wait(&empty[i], static_cast<uint32_t>(fills - 1) & 1u);
          }
        }
        mbar_wait(&eempty[es], eph ^ 1u);
        uint8_t* slot = ring + es * L.eslot;
        mbar_expect_tx(&efull[es], e_bytes);
        for (int bx = 0; bx < b.HW / 64; ++bx)
          tma_load_2d(slot + bx * ebox, &map_e, &efull[es], hs * b.HW + bx * 64, c * KV, pol_e);
        advance(es, eph, static_cast<int>(L.estages));
        PROBE(0, 100000 + j);
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the loops; each MMA / commit is issued by one
    // elected lane inside the asm (mma_bf16_warp: no per-MMA waterfall), and
    // the shared-memory descriptors are built once per stage and advanced by
    // constant offsets (sdesc_add).  Single-thread issue with per-MMA
    // descriptors cost ~120-150 cycles per UTCHMMA (tools/mma_rate*.cu) --
    // at N = 32 slower than the E stream delivers its 64-KB stages.
    const uint32_t idesc_w = idesc_bf16(kTileRows, N, false, false);
    // E phase: with b.stack the hi and lo P tiles (rows [0, N) and [N, 2N) of
    // one SW64 tile) are ONE B operand of 2N rows -- one MMA per k-step
    // writes E.hi into columns [0, N) and E.lo into [N, 2N) of the sub-tile,
    // so the E tile (A) is read from shared memory once instead of twice
    const int NE = b.stack ? 2 * N : N;
    const uint32_t idesc_e = idesc_bf16(128, NE, /*a MN-major*/ true, /*b K-major*/ false);
    int stage = 0;
    uint32_t phase = 0;
    for (int t = 0; t < ntiles; ++t) {
      const int buf = t & 1;
      const uint32_t use = static_cast<uint32_t>(t >> 1);
      // a tile of more than 128 rows: a second UMMA over rows [128, 256) of each chunk
      const bool two = tile_unit(sc0, nunits, ntiles, t + 1) - tile_unit(sc0, nunits, ntiles, t) > 4;
      mbar_wait(&tempty[buf], (use & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t d = tmem_base + static_cast<uint32_t>(buf * 2 * N);
      for (int kc0 = 0; kc0 < a.num_kc; kc0 += 2) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (tr != nullptr && t == 0 && kc0 == 0) tr[1] = globaltimer_ns();
        const uint32_t slot = smem_u32(ring + stage * L.wslot);
        const uint64_t a0 = sdesc_sw128(slot, 16, 1024), b0 = sdesc_sw128(slot + kWBytes, 16, 1024);
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int k = 0; k < kKChunk / 16; ++k) {
            const uint64_t bd = sdesc_add(b0, j * hchunk + k * 32);
            const uint32_t acc = ((kc0 + j) != 0 || k != 0) ? 1u : 0u;
            mma_bf16_warp(d, sdesc_add(a0, j * kChunkSpace + k * 32), bd, idesc_w, acc);
            if (two) mma_bf16_warp(d + N, sdesc_add(a0, j * kChunkSpace + kTileRows * 128 + k * 32), bd, idesc_w, acc);
          }
        mma_commit_warp(&empty[stage]);
        advance(stage, phase, a.stages);
      }
      mma_commit_warp(&tfull[buf]);
      if (lane == 0) PROBE(1, 1000 + t);
    }
    int ps = 0, es = 0;
    uint32_t pph = 0, eph = 0;
    const int nsub = b.nsub;  // <= 8 (HW <= 1024)
    for (int j = 0; j < n_all; ++j) {
      const bool own = j < n_own;
      // stack mode: ONE accumulator (relative to the per-row reference the P
      // producers choose); else own rows in set A, the other slabs' in set B
      const uint32_t set = (own || b.stack) ? 0u : kSetB;
      const bool first = (j == 0) || (j == n_own && !b.stack);
      if (lane == 0) PROBE(1, 100000 + j);
      mbar_wait(&pfull[ps], pph);
      if (lane == 0) PROBE(1, 200000 + j);
      mbar_wait(&efull[es], eph);
      if (lane == 0) PROBE(1, 300000 + j);
      tc_fence_after();
      if (tr2 != nullptr && j == 0) tr2[1] = globaltimer_ns();
      // A: [128 h x 16 v] = two 64-h boxes (LBO = box bytes), 8-v groups 1 KB apart (SBO);
      // B: P tile [N x 16 v] K-major SWIZZLE_64B (64-B rows, 8-row atoms of 512 B)
      const uint64_t a0 = sdesc_sw128(smem_u32(ring + es * L.eslot), ebox, 1024);
      const uint64_t bh0 = sdesc_swz(smem_u32(p_sm + ps * L.p_stage), 16, 512, 4);
#pragma unroll
      for (int k = 0; k < KV / 16; ++k) {
        const uint64_t bhi = sdesc_add(bh0, k * 32), blo = sdesc_add(bh0, p_half + k * 32);
#pragma unroll
        for (int sub = 0; sub < 8; ++sub) {
          if (sub < nsub) {
            const uint64_t ad = sdesc_add(a0, sub * 2 * ebox + k * 16 * 128);
            const uint32_t d = tmem_base + set + static_cast<uint32_t>(sub * NE);
            mma_bf16_warp(d, ad, bhi, idesc_e, (first && k == 0) ? 0u : 1u);
            if (!b.stack) mma_bf16_warp(d, ad, blo, idesc_e, 1u);
          }
        }
      }
      mma_commit_warp(&eempty[es]);
      mma_commit_warp(&pempty[ps]);
      if (b.stack && j == n_own - 1 && has_oth) mma_commit_warp(owndone);  // (rare) reference switch waits on it
      advance(es, eph, static_cast<int>(L.estages));
      advance(ps, pph, b.pstages);
    }
    mma_commit_warp(accfull);
    if (lane == 0) PROBE(1, 999999);
    if (tr2 != nullptr) {
      mbar_wait(accfull, 0);
      tr2[2] = globaltimer_ns();
    }
    __syncwarp();
  } else if (warp == 6) {
    // ------------------------------------------------------------ logits producer
    const uint64_t pol = policy_evict_last();  // flog chunks are read by the HS CTAs of the group
    int ps = 0;
    uint32_t pph = 0;
    if (n_all > 0) mbar_wait(own_ready, 0);
    fence_proxy_async_global();  // own generic-proxy flog writes -> TMA reads
    for (int j = 0; j < n_all; ++j) {
      if (j == n_own) {
        // other slabs of the group: wait for their W phase (group counter),
        // then m_oth[s] = max of their partial maxima
        if (lane == 0) {
          const volatile unsigned* cnt = b.grp_cnt + grp;
          uint32_t spins = 0;
          while (*cnt < static_cast<unsigned>(SPG)) {
            __nanosleep(64);
            if (++spins > (1u << 26)) __trap();
          }
          __threadfence();
          group_pass(b, grp, SPG);
        }
        __syncwarp();
        __threadfence();
        fence_proxy_async_global();
        for (int s = lane; s < N; s += kWarpThreads) {
          float mo = 0.f;
          if (s < a.M) {
            mo = neg_inf();
            const float4* pp = b.part1 + static_cast<long>(s) * b.grid1 + grp * SPG;
            for (int o = 0; o < SPG; ++o)
              if (o != q) mo = fmaxf(mo, __ldcg(&pp[o].x));
          }
          m_oth[s] = mo;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(oth_ready);
      }
      if (lane == 0) {
        mbar_wait(&fempty[ps], pph ^ 1u);
        mbar_expect_tx(&ffull[ps], f_bytes);
        tma_load_2d(f_sm + ps * L.f_stage, &map_f, &ffull[ps], chunk_at(j) * KV, 0, pol);
        PROBE(2, 100000 + j);
      }
      advance(ps, pph, b.pstages);
    }
    __syncwarp();
  } else if (warp < kEpiWarps) {
    // ------------------------------------------------------------ W phase: K1 epilogue
    grid_dep_wait();  // mask / credit ids of the previous step's commit visible
    if (a.wdur != nullptr && threadIdx.x == 0) t_start = globaltimer_ns();
    // record stats rows of this step (slot (epoch & 1) of a double-buffered record)
    float* recw = a.rec;
    if (a.rec_par > 0) recw += (*reinterpret_cast<const volatile unsigned*>(a.rec_ctl) & 1u) * a.rec_par;
    if (a.mask_snap != nullptr && blockIdx.x == 0)
      for (int s = threadIdx.x; s < a.M; s += kEpiThreads) a.mask_snap[s] = a.block_start ? 1 : a.mask[s];
    if (a.cids_snap != nullptr && blockIdx.x == 0)
      for (int e = threadIdx.x; e < a.M * a.K; e += kEpiThreads) {
        a.cids_snap[e] = a.block_start ? -1 : a.credit_ids[e];
        a.cval_snap[e] = a.block_start ? 0.f : a.credit_val[e];
      }
    if (a.credit_ids != nullptr && !a.block_start) {  // block start: no credited token yet
      const int stride = kStatWords + a.K;
      for (int e = threadIdx.x; e < a.M * a.K; e += kEpiThreads) {
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
    const uint64_t pol_flog = (a.xbits & 64) ? policy_evict_normal() : policy_evict_last();  // 64: old policy (A/B)
    const int stride = kStatWords + a.K;
    for (int t = 0; t < ntiles; ++t) {
      const int buf = t & 1;
      const uint32_t use = static_cast<uint32_t>(t >> 1);
      mbar_wait(&tfull[buf], use & 1u);
      tc_fence_after();
      const int trow0 = min(a.V_local, KV * tile_unit(sc0, nunits, ntiles, t));
      const int trows = min(a.V_local, KV * tile_unit(sc0, nunits, ntiles, t + 1)) - trow0;  // valid rows
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
          tmem_ld32(tmem_base + (static_cast<uint32_t>(warp * 32) << 16) +
                        static_cast<uint32_t>((buf * 2 + u) * N + g * 32),
                    x);
          if (valid && (a.xbits & 2) == 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = g * 32 + j;
              if (col < a.M) st_global_hint_f32(a.flog + static_cast<long>(col) * a.V_local + lv, x[j], pol_flog);
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
    if (tr != nullptr && threadIdx.x == 0) tr[2] = globaltimer_ns();
    if (a.wdur != nullptr && threadIdx.x == 0) a.wdur[blockIdx.x] = static_cast<unsigned>(globaltimer_ns() - t_start);
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
    for (int col = threadIdx.x; col < N; col += kEpiThreads) {
      float m = red[col * 3 + 0], l = red[col * 3 + 2];
      int ix = __float_as_int(red[col * 3 + 1]);
      for (int w = 1; w < kEpiWarps; ++w) {
        const float* r = red + (w * N + col) * 3;
        stat_combine(m, ix, l, r[0], __float_as_int(r[1]), r[2]);
      }
      if (col < a.M) {
        reinterpret_cast<float4*>(a.part)[static_cast<long>(col) * gridDim.x + role] =
            make_float4(m, __int_as_float(ix), l, 0.f);
        if (b.rec_acc != nullptr && n_own > 0) atomicMax(b.mx + col, f2ord(m));  // -> m_rank
        m_own[col] = m;
      } else {
        m_own[col] = 0.f;
      }
      if (b.stack) scB[col] = m_own[col];  // the E phase's reference (ref below), ordered by the barrier
      if (!has_oth) m_oth[col] = neg_inf();
    }
    // Publish: flog rows, captured credited logits and the partial of this
    // slab are complete (release) -> the group counter (other CTAs of the
    // group) and own_ready (this CTA's logits producer).
    __threadfence();
    fence_proxy_async_global();
    named_bar_epi();
    if (threadIdx.x == 0) {
      if (b.rec_acc != nullptr) atomicAdd(b.rcnt, 1u);  // W phases done (m_rank complete at gridDim.x)
      if (SPG > 1) {
        atomicAdd(&a.grp_cnt[grp], 1u);
        if (!has_oth) {  // waits for nobody: passes right away (after its own count)
          __threadfence();
          group_pass(b, grp, SPG);
        }
      }
      if (n_all > 0) mbar_arrive(own_ready);
    }

    // ------------------------------------------------------------ E phase: P producers
    const int tid = threadIdx.x;
    int ps = 0;
    uint32_t pph = 0;
    const int cpr = KV / 8;  // 16-B chunks per P row (4)
    // Stack mode: one accumulator, reference ref[s] per row = the own slab max;
    // the other slabs' rows use it too (their weights e^{f - m_own} may exceed
    // 1: exact in bf16 hi + lo and fp32) unless the other slabs' max exceeds
    // it by more than kRefGap nats -- then (practically never) the finished
    // own-row accumulation is rescaled in TMEM to the other slabs' max.
    constexpr float kRefGap = 32.f;
    float* ref = scB;  // (stack mode does not use set B's scale); = m_own, written before the barrier above
    for (int j = 0; j < n_all; ++j) {
      if (j == n_own) {
        mbar_wait(oth_ready, 0);
        if (b.stack) {
          if (tid == 0) misc[3] = 0u;
          named_bar_epi();
          for (int s = tid; s < N; s += kEpiThreads) {
            float r = (n_own > 0) ? m_own[s] : m_oth[s];
            if (n_own > 0 && s < a.M && m_oth[s] > m_own[s] + kRefGap) {
              r = m_oth[s];
              atomicOr(&misc[3], 1u);
            }
            ref[s] = r;
          }
          named_bar_epi();
          if (misc[3] != 0u) {  // rescale columns s of every sub-tile by e^{m_own - m_oth}
            mbar_wait(owndone, 0);
            tc_fence_after();
            const int NE = 2 * N;
            const uint32_t lb = tmem_base + (static_cast<uint32_t>(warp * 32) << 16);
            for (int sub = 0; sub < b.nsub; ++sub)
              for (int c0 = 0; c0 < NE; c0 += 32) {
                float x[32];
                tmem_ld32(lb + static_cast<uint32_t>(sub * NE + c0), x);
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) {
                  const int s = (c0 + jj) % N;
                  if (s < a.M && ref[s] != m_own[s]) x[jj] *= fexp(m_own[s] - ref[s]);
                }
                tmem_st32(lb + static_cast<uint32_t>(sub * NE + c0), x);
              }
            tc_fence_before();
            named_bar_epi();
          }
        }
      }
      const float* mref = b.stack ? ref : ((j < n_own) ? m_own : m_oth);
      const int c = chunk_at(j);
      mbar_wait(&ffull[ps], pph);
      mbar_wait(&pempty[ps], pph ^ 1u);
      const float* fch = reinterpret_cast<const float*>(f_sm + ps * L.f_stage);
      uint8_t* phi = p_sm + ps * L.p_stage;
      uint8_t* plo = phi + p_half;
      for (int u = tid; u < N * cpr; u += kEpiThreads) {
        const int s = u / cpr, cc = u - s * cpr;
        const int v0 = c * KV + cc * 8;
        float p[8];
        if (s < a.M && v0 < a.V_local) {
          const float4* src = reinterpret_cast<const float4*>(fch + s * KV + cc * 8);
          const float4 q0 = src[0], q1 = src[1];
          const float ms = mref[s];
          p[0] = fexp(q0.x - ms); p[1] = fexp(q0.y - ms); p[2] = fexp(q0.z - ms); p[3] = fexp(q0.w - ms);
          p[4] = fexp(q1.x - ms); p[5] = fexp(q1.y - ms); p[6] = fexp(q1.z - ms); p[7] = fexp(q1.w - ms);
        } else {
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) p[jj] = 0.f;
        }
        float r[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) r[jj] = p[jj] - __bfloat162float(__float2bfloat16_rn(p[jj]));
        const uint4 hi = make_uint4(pack_bf16x2(p[0], p[1]), pack_bf16x2(p[2], p[3]), pack_bf16x2(p[4], p[5]),
                                    pack_bf16x2(p[6], p[7]));
        const uint4 lo = make_uint4(pack_bf16x2(r[0], r[1]), pack_bf16x2(r[2], r[3]), pack_bf16x2(r[4], r[5]),
                                    pack_bf16x2(r[6], r[7]));
        // SWIZZLE_64B: 16-B chunk index XOR address bits [7, 9) (= row bits [1, 3))
        const uint32_t off = static_cast<uint32_t>(s) * 64u + ((static_cast<uint32_t>(cc) ^ ((s >> 1) & 3u)) << 4);
        *reinterpret_cast<uint4*>(phi + off) = hi;
        *reinterpret_cast<uint4*>(plo + off) = lo;
      }
      mbar_arrive(&fempty[ps]);
      fence_proxy_async();  // generic-proxy smem writes -> visible to tcgen05.mma
      mbar_arrive(&pfull[ps]);
      if (tid == 0) PROBE(3, 100000 + j);
      advance(ps, pph, b.pstages);
    }

    // reference rescales of the two accumulator sets (no MMA dependence)
    if (tid == 0) PROBE(4, n_all * 10000 + n_own * 10 + (has_oth ? 1 : 0));
    if (b.rec_acc != nullptr) {
      // record mode, while the MMA warp finishes the last chunks: m_rank = max
      // of every slab's max (complete once every W phase is done -- normally
      // long ago); the scales take the accumulator(s) from their reference
      // (ref / m_own / m_oth) to m_rank.  The first CTA here merges the rank's
      // statistics into the record (when the record leaves the rank).
      if (tid == 0) {
        uint32_t spins = 0;
        while (ld_acquire_gpu(b.rcnt) < gridDim.x) {
          __nanosleep(32);
          if (++spins > (1u << 26)) __trap();
        }
        misc[12] = (b.merge_stats && atomicAdd(b.rcnt + 1, 1u) == 0u) ? 1u : 0u;
      }
      named_bar_epi();
      for (int s = tid; s < N; s += kEpiThreads) {
        const float mr = (s < a.M) ? ord2f(__ldcg(b.mx + s)) : 0.f;
        if (b.stack) {
          scA[s] = (n_all > 0 && s < a.M) ? fexp(ref[s] - mr) : 0.f;
        } else {
          scA[s] = (n_own > 0 && s < a.M) ? fexp(m_own[s] - mr) : 0.f;
          scB[s] = (has_oth && s < a.M) ? fexp(m_oth[s] - mr) : 0.f;
        }
      }
      if (misc[12] != 0u) {
        // fixed-order (deterministic) merge of the slab partials: (m, v*, l, 0)
        // rows; the captured credited logits were written there in the W phase
        float* rs = b.rec_stats + ((b.rec_par > 0) ? (*reinterpret_cast<volatile unsigned*>(b.x.ctl) & 1u) * b.rec_par : 0);
        for (int s = warp; s < a.M; s += kEpiWarps) {
          float m = neg_inf(), l = 0.f;
          int ix = INT_MAX;
          const float4* src = reinterpret_cast<const float4*>(a.part) + static_cast<long>(s) * gridDim.x;
          for (int j0 = 0; j0 < static_cast<int>(gridDim.x); j0 += 32 * 8) {
            float4 p[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int j = j0 + lane + 32 * u;
              p[u] = (j < static_cast<int>(gridDim.x)) ? __ldcg(src + j)
                                                       : make_float4(neg_inf(), __int_as_float(INT_MAX), 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) stat_combine(m, ix, l, p[u].x, __float_as_int(p[u].y), p[u].z);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const float rm = __shfl_xor_sync(0xffffffffu, m, o);
            const int ri = __shfl_xor_sync(0xffffffffu, ix, o);
            const float rl = __shfl_xor_sync(0xffffffffu, l, o);
            stat_combine(m, ix, l, rm, ri, rl);
          }
          if (lane == 0)
            *reinterpret_cast<float4*>(rs + static_cast<long>(s) * b.rec_stride) =
                make_float4(m, __int_as_float(ix), l, 0.f);
        }
      }
    }
    for (int s = tid; s < N && b.rec_acc == nullptr; s += kEpiThreads) {
      const float mo = m_own[s], mt = m_oth[s];
      const float mg = fmaxf(mo, mt);
      if (b.stack) {  // the single accumulator is relative to ref[s]
        scA[s] = (n_all > 0 && s < a.M) ? fexp(ref[s] - mg) : 0.f;
      } else {
        scA[s] = (n_own > 0 && s < a.M) ? fexp(mo - mg) : 0.f;
        scB[s] = (has_oth && s < a.M) ? fexp(mt - mg) : 0.f;
      }
      if (hs == 0 && s < a.M) b.mref[static_cast<long>(grp) * a.M + s] = mg;
    }
  }

  // ------------------------------------------------------------ epilogue: partial rows
  // All 8 warps (the TMA / MMA / logits warps are idle by now): warps w and
  // w + 4 read the same TMEM lane quarter, so the two warp groups take half of
  // the hidden sub-tiles each.  TMEM [128 h lanes x 32 s] -> smem tile
  // [32 s][128 h] (the idle ring, double-buffered per group) -> coalesced
  // float4 rows of the [M][H] partial.
  asm volatile("bar.sync 3, %0;" ::"n"(kThreads) : "memory");  // scA / scB visible
  if (n_all > 0) {
    if (b.probe != nullptr) {
      uint32_t spins = 0;
      while (!mbar_try_wait(smem_u32(accfull), 0)) {
        if (++spins > (1u << 24)) {
          if (threadIdx.x == 0) {
            volatile int* o = b.probe + blockIdx.x * 64;
            for (int w = 0; w < 8; ++w) o[w] = prog[w];
            const int nb = 2 * a.stages + 4 + 4 * b.pstages + 3;
            for (int w = 0; w < nb && w < 28; ++w) {
              const uint64_t raw = *reinterpret_cast<volatile uint64_t*>(full + w);
              o[8 + 2 * w] = static_cast<int>(raw & 0xffffffffu);
              o[9 + 2 * w] = static_cast<int>(raw >> 32);
            }
            __threadfence_system();
          }
          __trap();
        }
      }
    } else {
      mbar_wait(accfull, 0);
    }
    tc_fence_after();
  }
  if (threadIdx.x == 0) PROBE(5, 1);
  unsigned long long t_epi = 0;
  if (tr2 != nullptr && threadIdx.x == 0) t_epi = globaltimer_ns();
  const bool recmode = b.rec_acc != nullptr;
  float* rec_acc = b.rec_acc;
  if (recmode && b.rec_par > 0) rec_acc += (*reinterpret_cast<volatile unsigned*>(b.x.ctl) & 1u) * b.rec_par;
  {
    const int wg = warp / 4, wq = warp % 4, tg = threadIdx.x % kEpiThreads;
    const int ng = N / 32;
    const int half = (b.nsub + 1) / 2;
    const int sub0 = (wg == 0) ? 0 : half, sub1 = (wg == 0) ? half : b.nsub;
    float* tile = reinterpret_cast<float*>(ring) + wg * 2 * (32 * 128);
    const int hbase = hs * b.HW;
    const uint64_t pol_part = policy_evict_last();  // kept in L2 for K34 (the weight streams are evict_first)
    const uint32_t lanebase = tmem_base + (static_cast<uint32_t>(wq * 32) << 16);
    const int NE = b.stack ? 2 * N : N;
    for (int sub = sub0; sub < sub1; ++sub) {
      for (int g = 0; g < ng; ++g) {
        float x[32];
        const uint32_t col = static_cast<uint32_t>(sub * NE + g * 32);
        if (n_own > 0 || (b.stack && n_all > 0)) {
          if (b.stack) {  // E.hi + E.lo (columns col and col + N), the single accumulator
            float y[32];
            tmem_ld32x2(lanebase + col, lanebase + col + N, x, y);
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) x[jj] = (x[jj] + y[jj]) * scA[g * 32 + jj];
          } else {
            tmem_ld32(lanebase + col, x);
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) x[jj] *= scA[g * 32 + jj];
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) x[jj] = 0.f;
        }
        if (has_oth && !b.stack) {
          float y[32];
          if (b.stack) {
            float z[32];
            tmem_ld32x2(lanebase + kSetB + col, lanebase + kSetB + col + N, y, z);
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) y[jj] += z[jj];
          } else {
            tmem_ld32(lanebase + kSetB + col, y);
          }
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) x[jj] = fmaf(y[jj], scB[g * 32 + jj], x[jj]);
        }
        if (recmode) {  // L2 reductions straight from the registers: 32 lanes = 128 contiguous bytes per row
          float* dst = rec_acc + hbase + sub * 128 + wq * 32 + lane;
#pragma unroll
          for (int jj = 0; jj < 32; ++jj)
            if (g * 32 + jj < a.M) atomicAdd(dst + static_cast<long>(g * 32 + jj) * a.H, x[jj]);
          continue;
        }
        if (b.part_tma) {
          // fp16 rows [32 s][128 h] in their own 8-KB tile (the idle ring:
          // one tile per (sub-tile, column group) of the warpgroup, never
          // reused, so no wait before the next pass), stored by one TMA
          // box per pass -- the thread-store version (fp32 tile, 8 B per
          // thread store) took ~5 us per CTA after the last E MMA
          __half* th = reinterpret_cast<__half*>(ring) + (wg * half * ng + (sub - sub0) * ng + g) * (32 * 128);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) th[jj * 128 + wq * 32 + lane] = __float2half_rn(x[jj]);
          fence_proxy_async();  // generic-proxy smem writes -> the TMA store
          if (wg == 0) {
            asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
          } else {
            asm volatile("bar.sync 2, %0;" ::"n"(kEpiThreads) : "memory");
          }
          if (tg == 0) {  // rows past M are outside the map: not written
            tma_store_3d(&map_p, th, hbase + sub * 128, g * 32, grp, pol_part);
            bulk_commit_group();
          }
          continue;
        }
        float* t = tile + (((sub - sub0) * ng + g) & 1) * (32 * 128);  // two tiles: one barrier per pass
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) t[jj * 128 + wq * 32 + lane] = x[jj];
        if (wg == 0) {
          asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
        } else {
          asm volatile("bar.sync 2, %0;" ::"n"(kEpiThreads) : "memory");
        }
        for (int u = tg; u < 32 * 32; u += kEpiThreads) {
          const int row = u >> 5, c4 = u & 31;
          const int s = g * 32 + row;
          if (s < a.M && (a.xbits & 16) == 0)  // xbits 16: measurement only, partial stores skipped
            st_global_hint_v2(b.part + (static_cast<long>(grp) * a.M + s) * a.H + hbase + sub * 128 + c4 * 4,
                              pack_half4(*reinterpret_cast<const float4*>(t + row * 128 + c4 * 4)), pol_part);
        }
      }
    }
  }
  if (recmode) __threadfence();  // this CTA's reductions before its count below
  if (!recmode && b.part_tma && threadIdx.x % kEpiThreads == 0) bulk_wait_group_all();  // partials written
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc(tmem_base, 512);
  if (a.wdur != nullptr && threadIdx.x == 0)  // whole-CTA duration (calibration objective)
    a.wdur[gridDim.x + blockIdx.x] = static_cast<unsigned>(globaltimer_ns() - t_start);
  // trace: K2-slot exit = end of the partial write-out / reductions, K1-slot exit = kernel exit
  if (tr2 != nullptr && threadIdx.x == 0) {
    tr2[0] = t_epi;  // (measurement) write-out start
    tr2[3] = globaltimer_ns();
  }
  if (recmode && threadIdx.x == 0 && atomicAdd(b.rcnt + 2, 1u) == gridDim.x - 1) {
    // the last CTA: every CTA has read m_rank and counted its reductions --
    // reset the self-resetting words for the next step, then (peer exchange)
    // raise this rank's flag in every peer
    b.rcnt[0] = 0u;
    b.rcnt[1] = 0u;
    b.rcnt[2] = 0u;
    for (int s = 0; s < a.M; ++s) b.mx[s] = 0u;
    if (b.x.peers != nullptr) {
      const unsigned epoch = *reinterpret_cast<volatile unsigned*>(b.x.ctl);
      const unsigned par = epoch & 1u;
      __threadfence_system();
      for (int j = 0; j < b.x.world; ++j) {
        unsigned* f = reinterpret_cast<unsigned*>(b.x.peers[j] + b.x.flags_off) + par * b.x.world +
                      (b.x.loopback ? j : b.x.rank);
        // relaxed: the fence above orders the record before these flags (one
        // release per flag serialised G system-scope round trips: ~2 us each)
        asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch + 1u) : "memory");
      }
    }
  }
  if (tr != nullptr && threadIdx.x == 0) tr[3] = globaltimer_ns();
}

}  // namespace

size_t k12_smem_bytes(int N, int HW, int stages, int pstages, int slab_rows_max, int emin) {
  const Layout L = make_layout(N, HW, stages, pstages, slab_rows_max, emin);
  if (L.estages < 2u) return ~size_t(0) >> 1;  // the E ring needs >= 2 slots: never fits
  return L.total + 1024;
}

int k12_blocks_per_sm(size_t smem) {
  if (ensure_func_smem(reinterpret_cast<const void*>(k12_proj_smooth), smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k12_proj_smooth, kThreads, smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

cudaError_t launch_k12(const CUtensorMap& map_w, const CUtensorMap& map_w32, const CUtensorMap& map_h,
                       const CUtensorMap& map_e, const CUtensorMap& map_f, const CUtensorMap& map_p, const K1Args& a,
                       const K2Args& b, int grid, size_t smem, cudaStream_t st, bool pdl) {
  {
    const cudaError_t e = ensure_func_smem(reinterpret_cast<const void*>(k12_proj_smooth), smem);
    if (e != cudaSuccess) return e;
  }
  return launch_ex(k12_proj_smooth, dim3(grid), dim3(kThreads), smem, st, pdl, map_w, map_w32, map_h, map_e, map_f,
                   map_p, a, b);
}

}  // namespace dinfer
