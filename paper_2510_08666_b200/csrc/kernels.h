// kernels.h -- internal launch interface between the C-ABI layer (dinfer_api.cu)
// and the step kernels.  Not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dinfer {

constexpr int kWarpThreads = 32;
constexpr int kKChunk = 64;        // bf16 elements per 128-B swizzled row
constexpr int kTileRows = 128;     // UMMA M (vocab rows per tile)
constexpr int kRowGran = 8;        // vocab-row granularity of the K1 partition
constexpr int kMaxCreditEnt = 1024;  // per-CTA credited (position, slot) entries
constexpr int kStatWords = 4;
constexpr int kTraceK34 = 64;     // K34 blocks traced (DINFER_TRACE)
constexpr int kChunkRows12 = 32;  // K12: vocab rows per E chunk (two UMMA K steps)

// Launch helper: optional programmatic dependent launch (PDL) attribute.
template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                      Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// cudaFuncSetAttribute applies to the CURRENT device only: the dynamic
// shared-memory limit (and optionally the carveout) of each kernel is raised
// per (kernel, device) pair, under a mutex (host threads may create contexts
// concurrently, on different devices).  Implemented in dinfer_api.cu.
cudaError_t ensure_func_smem(const void* fn, size_t smem, int carveout_pct = -1);

// Device-side sticky error bits (dinfer_sync reads and clears them).
enum : int { kErrCreditEntOverflow = 1, kErrCreditSlotsFull = 2, kErrCreditInvalid = 4 };

// ---------------------------------------------------------------- K1
struct K1Args {
  int M, N, H, K;          // positions, MMA N (>= M, %16), hidden, credit slots
  int V_local, v_offset;
  int num_kc;              // H / 64
  int h_resident;          // 1: whole hidden block resident in smem
  int stages;
  int slab_rows_max;       // max rows of any CTA's slab (credit head table size)
  const uint8_t* mask;     // [M]
  const int32_t* credit_ids;  // [M][K] or nullptr
  int VG, SPG, nchunks;     // vocab groups (K2-chunk aligned) x slabs per group = grid
  int chunk_rows;          // K2 chunk rows (group boundaries are multiples of it)
  float* part;             // [M][grid] float4 per-CTA (m, idx, l, 0), column-major
  unsigned* grp_cnt;       // [VG] slabs completed per group (K2 waits, resets), or nullptr
  float* rec;              // [M][4+K] rank record: only fcred (captured credited logits) is written
  long rec_par;            // > 0: `rec` is double-buffered, slot (rec_ctl[0] & 1) at rec + slot * rec_par
  const unsigned* rec_ctl; //      (the exchange epoch, advanced by K34)
  float* flog;             // [M][V_local] raw logits for K2, or nullptr
  uint8_t* mask_snap;      // [M] copy of the step-start mask (written by CTA 0), or nullptr
  int32_t* cids_snap;      // [M][K] copy of the step-start credit slots (f4), or nullptr
  float* cval_snap;
  const float* credit_val; // [M][K] (read for the snapshot)
  int* err;
  unsigned long long* trace;  // optional [grid][5]: globaltimer ns start, first W stage, last tile done, exit; smid
  // K12 calibrated partition (dinfer_balance; nullptr = the even one): CTA b
  // plays role role_of[b] (group role / SPG, slab role % SPG) and, with
  // SPG == 2, group g's rows split at chunk split[g]; wdur[b] <- W-phase ns.
  const int* role_of;
  const int* split;
  unsigned* wdur;
  // K1 calibrated slabs (stats-only contexts, VG == 1; nullptr = even):
  // CTA b covers rows [slab_start[b], slab_start[b+1]) (8-row multiples)
  const int* slab_start;
  // K12 calibrated vocab groups (nullptr = even): group g = chunks [grp_start[g], grp_start[g+1])
  const int* grp_start;
  int block_start;         // params.block_start: mask / credit inputs not read (all undecided, slots empty)
  int npre;                // K12: W stages issued before the dependency wait (0 = the whole ring; tuning)
  int xbits;               // K12 measurement-only experiments (env DINFER_K12_X; 0 in the product):
                           //   1 no hidden loads, 2 no flog stores, 4 W evict_normal, 8 E evict_normal
};
size_t k1_smem_bytes(int N, int H, int stages, int h_resident, int slab_rows_max);
cudaError_t launch_k1(const CUtensorMap& map_w, const CUtensorMap& map_w8, const CUtensorMap& map_w32,
                      const CUtensorMap& map_h, const K1Args& a, int grid, size_t smem, cudaStream_t st, bool pdl);

// ---------------------------------------------------------------- K1b (M > 256)
struct K1bArgs {
  int M, H, V_local, v_offset;
  int VG;                  // vocab groups (record rows per position)
  int stages;
  float* part;             // [VG][M] float4 (m, v* bits, l, 0) -- K3 reads it as VG "ranks"
};
size_t k1b_smem_bytes(int stages);
cudaError_t launch_k1b(const CUtensorMap& map_h, const CUtensorMap& map_w, const K1bArgs& a, int grid, size_t smem,
                       cudaStream_t st, bool pdl);

// Peer-memory record exchange (world > 1, dinfer_exchange_open): every rank
// keeps its own record double-buffered by epoch parity in its exchange buffer
// (IPC-shared); the kernel that completes it raises this rank's flag
// (= epoch + 1) in every peer's buffer, and K34 reads the peers' records
// in place (NVLink loads).  `peers` == nullptr: no flags to raise.
struct XArgs {
  float* const* peers;     // [world] device pointers to the ranks' exchange buffers, or nullptr
  int world, rank;
  long flags_off;          // word offset of the flags [2][world] in an exchange buffer
  unsigned* ctl;           // local control words: [0] epoch (advanced by K34), [1] finished blocks
  int loopback;            // measurement: peers are this GPU's own buffer, all `world` flags raised
};

// Rank record finalize (K1 / K1 -> K2 sharded and split-phase paths):
//   stats: rec[s] = merge of K1's per-slab partials (fixed order);
//   acc (if part2): rec_acc[s,:] = sum_g part2[g][s,:] * e^{m_g - m_rank}.
struct RecArgs {
  int M, H, grid1, VG, rec_stride;
  const float4* part1;
  const uint16_t* part2;   // [VG][M][H] fp16 or nullptr
  const float* mref;       // [VG][M]
  float* rec;              // stats rows (slot 0 when par_words > 0)
  long acc_off;            // words from a record's start to its acc part
  long par_words;          // > 0: double-buffered record, slot (epoch & 1) at rec + par * par_words
  XArgs x;
};

// ---------------------------------------------------------------- K2
struct K2Args {
  int M, N, H, V_local;
  int HW, nsub;            // hidden columns per CTA (128 .. 1024), HW/128
  int KV;                  // vocab rows per chunk: 64 (P tile SW128) or 32 (SW64, for HW = 1024)
  int HS, VG;              // H/HW slices, vocab groups
  int nchunks;             // ceil(V_local / KV)
  int stages, pstages;
  const float* flog;       // [M][V_local]
  const float4* part1;     // K1 partials [M][grid1]
  int grid1, SPG;          // K1 slabs, slabs per vocab group
  unsigned* grp_cnt;       // [VG] K1 slabs done per group
  unsigned* grp_pass;      // [VG] K2 CTAs past the wait (the last resets both)
  float* mref;             // [VG][M] out: per-group reference max m_g (acc is relative to it)
  uint16_t* part;          // [VG][M][H] fp16 (common.cuh: pack_half4)
  unsigned long long* trace;  // optional [grid][5]: globaltimer ns start, first E stage, MMAs done, exit; smid
  volatile int* probe;     // K12 diagnostics (env DINFER_K12_PROBE): [grid][8] progress words in mapped host memory
  int stack;               // K12: hi / lo P tiles stacked into one 2N-column MMA (TMEM nsub x 2N per set)
  int emin;                // K12: minimum E-ring depth (the ring is sized for it)
  int part_tma;            // K12 world-1 epilogue: fp16 partials stored by TMA (map_p) instead of thread stores
  // K12 record mode (rec_acc != nullptr): instead of per-group fp16 partials,
  // every CTA rescales its smoothing accumulator to the rank max m_rank (the
  // max of all slab maxima, gathered with atomicMax once every W phase is
  // done) and adds it into ONE fp32 record [M][H] with L2 reductions
  // (red.global.add.f32) -- the cross-CTA reduction overlaps the CTAs' finish
  // spread, and K34 reads one record instead of VG partials.
  float* rec_acc;          // record acc (slot 0 when rec_par > 0), relative to m_rank
  float* rec_stats;        // record stats rows (slot 0), stride rec_stride: (m, v*, l, 0, fcred[K])
  long rec_par;            // > 0: double-buffered by epoch parity (peer exchange), slot stride in words
  int rec_stride;
  int merge_stats;         // the first CTA to finish merges the slab statistics into the stats rows
  unsigned* mx;            // [M] ordered-uint max of the slab maxima (self-resetting)
  unsigned* rcnt;          // [4] W phases done, finish ticket, CTAs done (self-resetting)
  XArgs x;                 // flags raised by the last CTA (peer exchange)
};
size_t k2_smem_bytes(int N, int HW, int KV, int stages, int pstages);
cudaError_t launch_k2(const CUtensorMap& map_e, const CUtensorMap& map_f, const K2Args& a, size_t smem,
                      cudaStream_t st, bool pdl);

// ---------------------------------------------------------------- K12 (K1 + K2 fused, N <= 64)
// Uses K1Args (W phase; VG x SPG slabs at 16-row chunk granularity,
// nchunks / chunk_rows in 16-row chunks) and K2Args (E phase; HS == SPG
// hidden slices of HW columns, pstages logits / P ring depth; stages unused).
size_t k12_smem_bytes(int N, int HW, int stages, int pstages, int slab_rows_max, int emin = 0);
// Co-resident K12 CTAs per SM at this shared-memory size (K12 CTAs of a vocab
// group wait for each other's W phase, so the whole grid must be resident).
int k12_blocks_per_sm(size_t smem);
cudaError_t launch_k12(const CUtensorMap& map_w, const CUtensorMap& map_w32, const CUtensorMap& map_h,
                       const CUtensorMap& map_e, const CUtensorMap& map_f, const CUtensorMap& map_p, const K1Args& a,
                       const K2Args& b, int grid, size_t smem, cudaStream_t st, bool pdl);

cudaError_t launch_rec_finalize(const RecArgs& a, cudaStream_t st, bool pdl);

// ---------------------------------------------------------------- K3
struct K3Args {
  int B, S, K, world;
  long V_total;            // credit ids outside [0, V_total) or negative credit values set kErrCreditInvalid
  int block_start, mask_id;  // params.block_start: state inputs not read; mask / tokens / slots all written
  const float4* part1;     // G = 1: K1 per-slab partials [M][grid1] (stats merged here), else nullptr
  int grid1;
  const float* recs;       // world records, `rec_words` apart (stats used when part1 == nullptr; fcred always)
  long rec_words;
  // peer exchange (pull, rpar > 0): record r is at rpv[r] + (epoch & 1) * rpar (overrides recs);
  // the pointers travel by value (no dependent load before the records)
  float* rpv[8];
  long rpar;
  const float* const* rb;  // (device, set by the kernel) base of record r, r < world
  int rec_stride;          // 4 + K
  uint8_t* mask;
  int32_t* tokens;
  int32_t* credit_ids;
  float* credit_val;
  uint8_t* committed;
  float* stats;            // [M][4] or nullptr
  float* ml;               // [M][2] merged (m, l) for K4
  float4* sel;             // [M] per-position (p~, v~ bits, undecided, 0) from the phase-1 CTAs
  int* row_cnt;            // [B] phase-1 CTAs arrived per batch row (zero between steps)
  int decoder, runs_after_hi, use_credit;
  int inclusive;           // thresholds compare '>=' instead of '>' (reading c1)
  float tau, theta_hi, theta_lo, c_alpha, c_beta, c_gamma;
  unsigned long long* trace;  // DINFER_TRACE: blocks < kTraceK34 stamp [entry, deps, phase1, end, smid]
  int H;
  const uint16_t* E;       // [V_local][H] bf16 (next-input embedding of committed rows) or nullptr
  uint16_t* emb;           // [M][H] bf16 next-iteration input embedding (f2) or nullptr
  int* rowdone;            // [M] smoothing blocks done per row (phase 2 waits, then resets)
  // Peer-memory exchange: the kernel waits until every rank's flag for this
  // epoch is up, reads the ranks' records of slot (epoch & 1) in place, and
  // its last block advances the epoch.
  const unsigned* xflags;  // [2][world] in the local exchange buffer, or nullptr
  unsigned* xctl;          // [0] epoch, [2] finished K34 blocks
  const float* pdev;       // optional device copy of the numeric params [tau, theta_hi, theta_lo,
                           // c_alpha, c_beta, c_gamma, alpha_t] (overrides the values above; lets a
                           // captured CUDA graph run with per-step schedules)
  int* err;
};


// ---------------------------------------------------------------- K4
struct K4Args {
  int M, H;
  // smoothing accumulators: either the world rank records (rec_mode: acc at
  // record + acc_off, relative to the record's m; rec_unit: ONE record
  // relative to the merged m itself, scale 1 -- world-1 K12 record mode) or
  // fp16 per-group partials (acc_h, relative to m_part)
  int rec_mode, rec_unit;
  long acc_off;
  float* zero_acc;         // record acc [M][H] to zero after the step (K12 record mode), or nullptr
  long zero_par;           // > 0: zero slot ((epoch & 1) ^ 1) of a double-buffered record instead
  const uint16_t* acc_h;   // fp16 partials (K2 output) at acc_h + p*acc_stride
  long acc_stride;
  int nparts;
  const float* m_part;     // m of partial p, row s at m_part[p*m_stride + s*m_rowstride]
  long m_stride;
  int m_rowstride;
  const uint8_t* mask_start;  // [M] mask at step start (snapshot; the selection blocks rewrite `mask`)
  const uint16_t* e_mask;  // [H] bf16
  float alpha_t;
  float* out;              // [M][H]
  const uint16_t* E;       // [V_local][H] bf16, with emb
  uint16_t* emb;           // [M][H] bf16 next-iteration input embedding or nullptr: E[token] for rows
                           // decided at step start, bf16(e_{t+1}) for the others (committed rows are
                           // then overwritten with E[v~] by the selection block)
  const int32_t* tokens;   // [M] (rows decided at step start are stable during the step)
  int* rowdone;            // [M]
  const int32_t* cids0;    // credit-fused smoothing (f4): step-start credit snapshot [M][K], or nullptr
  const float* cval0;
};
// K3 + K4 in one launch (a4 == nullptr: selection only)
cudaError_t launch_k34(const K3Args& a3, const K4Args* a4, cudaStream_t st, bool pdl);

// ---------------------------------------------------------------- generation loop (gen_loop.cu)
struct GenArgs {
  int B, S, L, P, K, nblocks;   // rows, block size, row length, prompt length, credit slots
  int mask_id, eos_id, early, decoder, use_smooth, use_credit, max_forwards;
  float tau_target;
  int tau_decay;
  float a_init, a_growth, a_preset;
  float base[8];                // step params [tau, theta_hi, theta_lo, c_alpha, c_beta, c_gamma, alpha_t, 0]
  int32_t* X;                   // [B][L] token rows (caller's, in/out)
  uint8_t* mask;                // block-local state the step runs on: [B][S]
  int32_t* tokens;              // [B][S]
  int32_t* cids;                // [B][S][K]
  float* cval;                  // [B][S][K]
  float* pdev;                  // [8] per-iteration step params (read by K34)
  int* st;                      // [4 + B]: block, t, F, truncated, row_done[B]
  int32_t* out;                 // [B + 2]: T[b], F, truncated (caller's)
  const uint16_t* hsrc;         // model stand-in: [hsrc_iters][M][H] bf16
  long hsrc_iters, MH;
  uint16_t* hbuf;               // [M][H] the step's hidden input
};
cudaError_t launch_gen_init(const GenArgs& a, cudaGraphConditionalHandle h, cudaStream_t st);
// host-buffer staging (stage.cu): zero-copy kernel copies of two 16-B aligned
// segments; `in`: trigger dependents at entry (host -> device inputs)
cudaError_t launch_stage_copy(const void* src0, void* dst0, size_t bytes0, const void* src1, void* dst1,
                              size_t bytes1, bool in, cudaStream_t st, bool pdl);
cudaError_t launch_block_reset(uint8_t* mask, int32_t* tokens, int32_t* cids, float* cval, int M, int K, int mask_id,
                               cudaStream_t st, bool pdl);
cudaError_t launch_gen_control(const GenArgs& a, cudaGraphConditionalHandle h, cudaStream_t st, bool pdl);
cudaError_t launch_gen_hidden(const GenArgs& a, int grid, cudaStream_t st);

}  // namespace dinfer
