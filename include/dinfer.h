/*
 * dinfer.h -- C ABI of the B200-native denoise-and-commit step of dInfer
 * (arXiv 2510.08666).  One call = one iteration of the inner `while` loop of
 * Algorithm 1 on the decode side:
 *
 *   logits = hidden x W_vocab^T            (never materialised in HBM
 *                                            for the statistics)
 *   credit update + fuse (App. B.2), threshold or
 *   hierarchical (App. B.1) commit rule, commit,
 *   iteration smoothing e_{t+1} = e_mask + alpha_t * softmax(z) W_emb
 *   (App. A.1) for positions still masked.
 *
 * The vocabulary may be sharded over `world` GPUs (contiguous rows of W_vocab
 * and W_emb); each rank builds one record (statistics + smoothing accumulator)
 * per step inside the producing kernel and the ranks exchange records over
 * peer memory (dinfer_exchange_open: every rank reads its peers' records in
 * place over NVLink once their flags are up) or, without opened peer
 * buffers, by one NCCL allgather; every rank then runs the identical combine,
 * so decode state stays replicated and bit-identical.
 *
 * Conventions (all entry points):
 *  - Every pointer is CALLER-OWNED; the library never frees or retains it
 *    beyond the call.  "device" pointers are CUDA global memory on the ctx's
 *    device; "host" pointers are ordinary (ideally pinned) host memory.
 *  - bf16 tensors are passed as `const uint16_t*` holding bf16 bit patterns.
 *  - Layouts are row-major and dense.  Flattened position index i = b*S + s.
 *  - Host-side validation is synchronous and has no side effects; on error
 *    nothing is enqueued.  Device work is asynchronous on the ctx stream, with
 *    no host synchronisation and no allocation (CUDA-Graph capturable), except
 *    dinfer_step_host and dinfer_sync which synchronise by definition.
 *  - Asynchronous faults (CUDA, NCCL, device-checked preconditions such as a
 *    full credit slot table) surface through dinfer_sync.
 *  - Readings of the paper's silent points (strict '>' thresholds, lowest-id
 *    argmax ties, fallback commit, run-based hierarchical rule, raw-softmax
 *    smoothing, ...) are listed in DESIGN.md "Readings" (c1..c20).
 */
#ifndef DINFER_H
#define DINFER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dinfer_ctx dinfer_ctx;

typedef enum {
  DINFER_OK = 0,
  DINFER_ERR_ARG = 1,         /* null / out-of-range argument                      */
  DINFER_ERR_SHAPE = 2,       /* inconsistent or unsupported shape / alignment     */
  DINFER_ERR_CUDA = 3,        /* CUDA runtime error                                 */
  DINFER_ERR_NCCL = 4,        /* NCCL error                                         */
  DINFER_ERR_NOMEM = 5,       /* device allocation failed                           */
  DINFER_ERR_UNSUPPORTED = 6, /* feature not available in this ctx / build          */
  DINFER_ERR_DEVICE = 7       /* device-checked precondition violated (sticky)      */
} dinfer_status;

enum { DINFER_DEC_THRESHOLD = 0, DINFER_DEC_HIERARCHICAL = 1 };

/* Problem shape, fixed at create time.
 *   B, S      batch rows and block size; M = B*S positions, 1 <= S <= 1024,
 *             M <= 256 (the HBM-bound swap-AB path; larger M is UNSUPPORTED).
 *   H         hidden size, multiple of 128.
 *   K         credit slots per position, >= 1 (K >= iterations per block is
 *             enough for an exact credit table).
 *   V_total   full vocabulary; V_local rows live on this rank starting at
 *             global id v_offset; V_local % 8 == 0, V_local * world == V_total.
 *   world, rank   vocab shards (1..8) and this rank.
 *   smooth_capable  1 to allocate the smoothing workspace (required for
 *             params.use_smooth).                                              */
typedef struct {
  int32_t B, S, H, K;
  int64_t V_total, V_local, v_offset;
  int32_t world, rank;
  int32_t smooth_capable;
} dinfer_shape;

/* Per-step parameters (host struct, read synchronously).
 *   decoder      DINFER_DEC_THRESHOLD: commit {undecided s : p~_s > tau}
 *                (strict '>', reading c1); DINFER_DEC_HIERARCHICAL:
 *                commit {p~ > theta_hi} plus, for every maximal run of
 *                undecided positions without such a commit, its best position
 *                if p~ > theta_lo (readings c8-c10; ties: nearest the
 *                run centre, then lower index).  Both: if nothing is committed
 *                in a batch row with undecided positions, commit its max-p~
 *                position (reading c2).  Thresholds in [0, 1].
 *   hier_runs_after_hi  0: runs from the mask at step start (reading c8 A);
 *                1: runs of positions left after the theta_hi commits (A').
 *   use_credit   credit decoding (App. B.2): C <- beta*C, C[v*] += p*^gamma for
 *                undecided positions, then f~ = f + c_alpha*log(1+C) and p~, v~
 *                from softmax(f~).  beta, gamma in (0,1); c_alpha >= 0.
 *   use_smooth   iteration smoothing with weight alpha_t >= 0.
 *   smooth_credit_fused  0: smooth with the raw softmax(z) (reading
 *                c13); 1: with the distribution the decoder decided on,
 *                softmax(f + c_alpha ln(1 + C)) -- exact, via the
 *                credited tokens' correction.  Requires use_credit,
 *                use_smooth, K <= 32 and world == 1 (else UNSUPPORTED).
 *   block_start  1: the step is the first iteration of a block (Alg. 1
 *                NextBlock; credit reset P:327): the mask / tokens /
 *                credit inputs are NOT read -- every position is undecided
 *                and every credit slot empty -- and all of them are written:
 *                mask = !committed, tokens = v~ where committed else mask_id,
 *                credit slots = this step's update from empty.  Same result
 *                as dinfer_block_reset + a step, one kernel boundary fewer.
 *   mask_id      token id of an undecided position (block_start only;
 *                in [0, V_total)).
 *   inclusive    0: threshold tests are strict, p~ > tau / theta (P:118
 *                "exceeds", reading c1; tau = 1 then commits exactly one
 *                position per step); 1: inclusive p~ >= tau / theta, the
 *                SPEC's reading (variant c1').  Both sides of every
 *                comparison are fp32 on the device.                         */
typedef struct {
  int32_t decoder;
  float tau;
  float theta_hi, theta_lo;
  int32_t hier_runs_after_hi;
  int32_t use_credit;
  float c_alpha, c_beta, c_gamma;
  int32_t use_smooth;
  float alpha_t;
  int32_t smooth_credit_fused;
  int32_t block_start;
  int32_t mask_id;
  int32_t inclusive;
} dinfer_params;

/* 128-byte NCCL unique id for world > 1 (rank 0 calls it and broadcasts). */
dinfer_status dinfer_get_unique_id(uint8_t out_id[128]);

/* Create a context on the current CUDA device.  `stream` is a cudaStream_t
 * (NULL = legacy default stream).  `nccl_unique_id`: 128 bytes from
 * dinfer_get_unique_id (all ranks the same) when world > 1, or NULL: then the
 * ctx has no communicator and only the split-phase calls
 * (dinfer_step_local / dinfer_step_combine) work for world > 1.  Allocates the
 * whole workspace once.  Errors: ARG, SHAPE, UNSUPPORTED, CUDA, NCCL, NOMEM. */
dinfer_status dinfer_create(const dinfer_shape* shape, const uint8_t* nccl_unique_id,
                            void* stream, dinfer_ctx** out);
void dinfer_destroy(dinfer_ctx* ctx);
dinfer_status dinfer_set_stream(dinfer_ctx* ctx, void* stream);

/* One denoise-and-commit iteration (device pointers, asynchronous).
 *   hidden      [B,S,H] bf16, identical on every rank.
 *   W_vocab     [V_local,H] bf16, this rank's rows of the LM head (nn.Linear).
 *   E           [V_local,H] bf16, this rank's rows of the input embedding
 *               W_emb; may be NULL iff !use_smooth.
 *   e_mask      [H] bf16 mask embedding; NULL iff !use_smooth.
 *   mask        [B,S] uint8 in/out, 1 = undecided; cleared where committed.
 *   tokens      [B,S] int32 in/out; written only at newly committed positions.
 *   credit_ids  [B,S,K] int32 in/out, -1 = empty slot; credit_val [B,S,K]
 *               float in/out.  Only rows undecided at step start change.
 *               May be NULL iff !use_credit.  Device-checked precondition
 *               (sticky, DINFER_ERR_DEVICE from dinfer_sync): every used
 *               slot of an undecided row has an id in [0, V_total) and a
 *               value >= 0, and a new id finds a free slot.
 *   committed   [B,S] uint8 out, 1 = committed by this step.
 *   smoothed    [B,S,H] float out: e_{t+1} for every row undecided at
 *               step start; it is meaningful for the rows still undecided
 *               after the commit (the caller feeds only those back).
 *               Rows decided at step start are untouched.  NULL iff !use_smooth.
 *   stats       [B,S,4] float out or NULL: (m = max logit, lse = log-sum-exp
 *               of the raw logits, p~ = confidence used by the decoder,
 *               v~ = committed/candidate id as int32 bits).
 * A batch row with no undecided position is a defined no-op (commits
 * nothing).  world > 1 requires a communicator (else UNSUPPORTED).           */
dinfer_status dinfer_step(dinfer_ctx* ctx, const uint16_t* hidden, const uint16_t* W_vocab,
                          const uint16_t* E, const uint16_t* e_mask, uint8_t* mask,
                          int32_t* tokens, int32_t* credit_ids, float* credit_val,
                          const dinfer_params* params, uint8_t* committed, float* smoothed,
                          float* stats);

/* dinfer_step plus the next iteration's model input (Fig. 3 /
 * PAPER.md:152): emb [B,S,H] bf16 device out,
 *   emb[s] = W_emb[tokens[s]]   for every position decided after this step
 *            (decided earlier, or committed now: its new token's row),
 *   emb[s] = bf16(e_{t+1}[s])   for positions still masked (= smoothed[s]).
 * Written by the same K34 launch (no extra kernel).  Requires use_smooth,
 * world == 1 (the embedding rows of committed tokens live on one rank) and
 * M <= 256; else UNSUPPORTED.  emb must be 16-byte aligned.                 */
dinfer_status dinfer_step_embed(dinfer_ctx* ctx, const uint16_t* hidden, const uint16_t* W_vocab,
                                const uint16_t* E, const uint16_t* e_mask, uint8_t* mask,
                                int32_t* tokens, int32_t* credit_ids, float* credit_val,
                                const dinfer_params* params, uint8_t* committed, float* smoothed,
                                float* stats, uint16_t* emb);

/* Same step with HOST per-step buffers (weights stay on device): copies
 * hidden and the decode state host->device, runs dinfer_step, copies the
 * state and outputs back, and synchronises the stream before returning.
 * Transfers: hidden (M*H*2 B) directly from hidden_h; the small state (the
 * numeric params, mask, tokens, credit table) packed through one pinned
 * staging block into one H2D copy; one D2H copy of the packed state +
 * committed + stats; smoothed (M*H*4 B) directly into smoothed_h.
 * On a single-rank ctx, or a sharded one whose exchange is peer memory
 * (dinfer_exchange_open / _loopback), with timing off, the whole sequence
 * (copies and kernels) is captured into a CUDA graph and replayed; the
 * numeric params (tau, theta_*, c_*, alpha_t) are read on device from the
 * packed block, so schedules never force a re-capture. The graph is keyed by
 * every pointer argument and by decoder / hier_runs_after_hi / use_credit /
 * use_smooth / stats_h nullness; the ctx keeps the 4 most recently used
 * graphs, so callers rotating a few buffers replay without re-capturing. Buffers the graph cannot capture (pageable
 * host memory) run the same sequence un-captured. hidden_h and smoothed_h
 * may be pageable; pinned buffers avoid a staging copy inside the driver,
 * and a pinned smoothed_h is written by the kernel directly (zero-copy; no
 * D2H copy for the M*H*4-byte output).  With a pinned hidden_h the two
 * host->device transfers become one staging kernel reading the mapped host
 * memory, chained ahead of the step by programmatic dependent launch (the
 * W stream starts under the PCIe reads), and the state goes back through a
 * second staging kernel writing the mapped pinned block. */
dinfer_status dinfer_step_host(dinfer_ctx* ctx, const uint16_t* hidden_h,
                               const uint16_t* W_vocab, const uint16_t* E,
                               const uint16_t* e_mask, uint8_t* mask_h, int32_t* tokens_h,
                               int32_t* credit_ids_h, float* credit_val_h,
                               const dinfer_params* params, uint8_t* committed_h,
                               float* smoothed_h, float* stats_h);

/* Calibrated vocab partition for the fused projection + smoothing kernel
 * (K12, hidden split in two slices).  Per-SM HBM streaming rates on B200
 * differ systematically (~100-123 us for equal W slabs at MoE shape; the
 * CTA -> SM placement of a full-machine launch is the same every launch),
 * so the finishing spread of equal slabs is exposed at the end of the step.
 * dinfer_balance runs `iters` (+1 warm-up) steps with the given weights on
 * scratch state, measures each CTA's time, pairs the slowest SM with the
 * fastest in each vocab group and splits the group's rows so both finish
 * together (W rows plus the group's E slice per CTA; 20..80 % bounds); later
 * steps use that partition (results are the same up to fp32 summation
 * order).  `mode` is the state the steps will run in, which shifts the per-SM
 * rates: DINFER_BALANCE_AFTER_FORWARD (0) -- each step follows an L2-dirtying
 * model forward (the calibration steps run after a 2x-L2 write);
 * DINFER_BALANCE_BACK_TO_BACK (1) -- steps follow each other directly (block
 * reset + step, PDL chain intact).  Synchronous; allocates scratch
 * temporarily.  On a stats-only context (smooth_capable = 0, params
 * without smoothing) it calibrates K1's slab sizes instead: rows per CTA
 * proportional to the measured per-SM rates (damped, 8-row units, at most
 * 1.3x the even slab).  UNSUPPORTED otherwise (two-kernel smoothing path,
 * M > 256); ARG for another mode.  dinfer_balance_reset restores the even
 * partition.                                                                */
#define DINFER_BALANCE_AFTER_FORWARD 0
#define DINFER_BALANCE_BACK_TO_BACK 1
dinfer_status dinfer_balance(dinfer_ctx* ctx, const uint16_t* hidden, const uint16_t* W_vocab,
                             const uint16_t* E, const uint16_t* e_mask, const dinfer_params* params,
                             int32_t iters, int32_t mode);
dinfer_status dinfer_balance_reset(dinfer_ctx* ctx);

/* Peer-memory exchange of the per-rank records (world > 1),
 * replacing the NCCL allgather: each rank keeps its record in its exchange
 * buffer, double-buffered by step parity (slot epoch & 1, so a rank one step
 * ahead never overwrites a slot a slower rank still reads).  The kernel that
 * completes it (K12's last CTA; the record finalize on the K1 paths) raises
 * this rank's flag (epoch + 1) in every peer's buffer; the select/commit
 * kernel waits for all flags of its epoch, reads the peers' records in place
 * over NVLink, zeroes its own consumed accumulator slot and advances the
 * epoch -- no host synchronisation, no NCCL launch, graph safe.
 * dinfer_exchange_handle: this ctx's exchange buffer as a 64-byte CUDA IPC
 * handle.  dinfer_exchange_open: `handles` = world handles back to back in
 * rank order (all ranks); after it, dinfer_step exchanges through peer memory
 * (no communicator needed).  Errors: ARG, UNSUPPORTED (world == 1), CUDA.  */
dinfer_status dinfer_exchange_handle(dinfer_ctx* ctx, uint8_t out_handle[64]);
dinfer_status dinfer_exchange_open(dinfer_ctx* ctx, const uint8_t* handles);
/* Measurement only: one rank of a `world`-way vocab shard on ONE GPU.  Every
 * "peer" is this ctx's own exchange buffer: each step raises all `world` flags
 * and the combine reads this rank's record `world` times, so the step runs
 * the kernels and moves the bytes of a real rank (minus the NVLink latency);
 * the combined results are NOT meaningful (the G records are copies of one
 * shard's).
 * Errors: ARG (already open), UNSUPPORTED (world == 1), CUDA.               */
dinfer_status dinfer_exchange_loopback(dinfer_ctx* ctx);

/* The same host-buffer step split in two: _async validates, stages the small
 * state, enqueues copies + step + result copies on the ctx stream and returns;
 * _wait synchronises the stream and unpacks mask / tokens / credit /
 * committed / stats into the host buffers given to _async (smoothed_h is
 * written by the device directly).  Lets the caller overlap its own host
 * work with the step, or time the step on the stream (CUDA events around
 * _async and its copies).  One pending call per ctx; _wait without a
 * pending _async returns ARG.                                               */
dinfer_status dinfer_step_host_async(dinfer_ctx* ctx, const uint16_t* hidden_h,
                                     const uint16_t* W_vocab, const uint16_t* E,
                                     const uint16_t* e_mask, uint8_t* mask_h, int32_t* tokens_h,
                                     int32_t* credit_ids_h, float* credit_val_h,
                                     const dinfer_params* params, uint8_t* committed_h,
                                     float* smoothed_h, float* stats_h);
dinfer_status dinfer_step_host_wait(dinfer_ctx* ctx);

/* Split phases (tests, caller-managed collectives).
 * dinfer_record_words: number of fp32 words of one rank's record:
 *   M*(4+K)  statistics: per row (m, v* as int32 bits (global id), l =
 *            sum_{v in shard} exp(f_v - m), 0, fcred[K] = raw logit of each
 *            credited token if this rank owns it else -inf), padded to a
 *            multiple of 4 words (the acc part stays 16-byte aligned)
 *   + M*H    (use_smooth only) acc[s,:] = sum_{v in shard} exp(f_v - m) E[v,:]
 *            (on the fused K12 path the sum over the shard's CTAs is taken with
 *            L2 reductions: reproducible to fp32 rounding order, not bitwise).
 * dinfer_step_local writes this rank's record to `record` (device, that many
 * words).  dinfer_step_combine reads `records` = `world` records back to back
 * (rank order) and performs the combine / credit / selection / commit /
 * smoothing exactly as dinfer_step.                                          */
size_t dinfer_record_words(const dinfer_ctx* ctx, int32_t use_smooth);
dinfer_status dinfer_step_local(dinfer_ctx* ctx, const uint16_t* hidden, const uint16_t* W_vocab,
                                const uint16_t* E, const uint8_t* mask, const int32_t* credit_ids,
                                const dinfer_params* params, float* record);
dinfer_status dinfer_step_combine(dinfer_ctx* ctx, const float* records, const uint16_t* e_mask,
                                  uint8_t* mask, int32_t* tokens, int32_t* credit_ids,
                                  float* credit_val, const dinfer_params* params,
                                  uint8_t* committed, float* smoothed, float* stats);

/* Block start: empty every credit slot (ids = -1, values = 0). */
dinfer_status dinfer_credit_reset(dinfer_ctx* ctx, int32_t* credit_ids, float* credit_val);

/* Block start (Alg. 1 NextBlock, with the credit reset of P:327)
 * as one kernel on the ctx stream: mask = 1 and tokens = mask_id for every
 * position, credit slots empty (credit_ids / credit_val both NULL to skip).
 * It lets the next dinfer_step start streaming W underneath it (programmatic
 * dependent launch).  Errors: ARG.                                          */
dinfer_status dinfer_block_reset(dinfer_ctx* ctx, uint8_t* mask, int32_t* tokens, int32_t* credit_ids,
                                 float* credit_val, int32_t mask_id);

/* Host schedule helpers.
 * alpha_t = min(init + growth*t, preset)
 * tau_t   = 1 - (1 - target)*min(t, decay_steps)/decay_steps,
 *           i.e. linear decay from 1.0 to target (reading c11);
 *           decay_steps <= 0 returns target.                                 */
float dinfer_alpha_schedule(float init, float growth, float preset, int32_t t);
float dinfer_tau_schedule(float target, int32_t t, int32_t decay_steps);

/* ---------------------------------------------------------------------------
 * Device-resident blockwise generation loop (Algorithm 1).
 *
 * dinfer_generate runs the block loop over the generation region
 * [prompt_len, L) of the token rows X [B][L] (device int32, in/out; mask_id
 * marks undecided positions), S positions per block, left to right, all B
 * rows in lockstep:
 *   for each block: credit table reset, t = 0;
 *     while any position of the block is undecided:
 *       hidden  <- the model's hidden states of this iteration (see below)
 *       params  <- tau_t (drives tau, or theta_hi for the hierarchical
 *                  decoder; reading c11), alpha_t, rest from `base`
 *       dinfer_step on the block; t += 1; F += 1
 *     early termination (reading c22): a row whose completed block
 *     holds eos_id is finished; its later blocks are filled with eos_id; the
 *     loop halts once every row is finished.
 * The whole loop is ONE CUDA graph (a conditional WHILE node around
 * {hidden, step kernels, bookkeeping kernel}) launched on the ctx stream: no
 * host synchronisation or data-dependent host control inside a generation.
 * Asynchronous like dinfer_step; results land in X and `out` (device int32
 * [B+2]: T_b = generated tokens before the first eos_id of row b (
 * gen_len if none), then F = forwards run, then 1 if max_forwards stopped
 * the loop early).  The graph is built on the first call and re-used while
 * the pointers and the configuration are unchanged.
 *
 * The model forward is not part of this library.  Its stand-in here is a
 * hidden-state source: iteration n (0-based, global) uses
 * hidden_src + min(n, hidden_iters-1)*B*S*H (bf16 [B][S][H] blocks, device),
 * copied into the step's hidden buffer -- the point where a real model's
 * captured forward is inserted.
 *
 * Constraints: (L - prompt_len) % S == 0 and > 0; ctx shape B, S as created;
 * world == 1; B <= 1024; mask_id, eos_id in [0, V_total).  `base` supplies the
 * decoder, theta_lo, credit constants and use_smooth/use_credit; its tau /
 * theta_hi / alpha_t are replaced per iteration by the schedules.
 * Smoothed embeddings of the last iteration stay in ctx-owned memory.      */
typedef struct {
  int32_t L;                 /* tokens per row (prompt + generation)          */
  int32_t prompt_len;        /* fixed input positions [0, prompt_len)         */
  int32_t mask_id, eos_id;
  int32_t early_termination;
  float tau_target;          /* tau_t = dinfer_tau_schedule(tau_target, t, tau_decay_steps) */
  int32_t tau_decay_steps;
  float alpha_init, alpha_growth, alpha_preset; /* alpha_t (used with smoothing) */
  int32_t max_forwards;      /* safety bound on F (>= 1)                        */
} dinfer_gen_config;

dinfer_status dinfer_generate(dinfer_ctx* ctx, const dinfer_gen_config* cfg, const dinfer_params* base,
                              const uint16_t* W_vocab, const uint16_t* E, const uint16_t* e_mask,
                              const uint16_t* hidden_src, int64_t hidden_iters, int32_t* X, int32_t* out);

/* ---------------------------------------------------------------------------
 * Vicinity KV-cache refresh (§2.3, App. D
 * P:368) on a synthetic single bidirectional attention layer: the KV-cache
 * manager of Algorithm 1 (K.ShouldUpdate / K.Update).
 *
 * Shape: L positions, hidden H = n_heads * d_head (d_head must be 128),
 * prefix_look / after_look (16 / 16 in the paper) and warmup_times (4).
 * Refresh region of a forward (readings c25-c27): for block [start, end) at
 * block-local iteration t, [0, L) while t < warmup_times or when `full`
 * (a completed block's full refresh), else
 * [start - prefix_look, end + after_look) clipped to [0, L).
 *
 * dinfer_kv_step (device pointers, asynchronous on the kv stream):
 *   X        [L,H] bf16 layer input of every position (this iteration)
 *   Wq/Wk/Wv [H,H] bf16 projections, nn.Linear layout [out, in]
 *   Kc, Vc   [L,H] bf16 caller-owned caches, updated IN PLACE on the region
 *            (bf16 of the fp32-accumulated projection); other rows untouched
 *   out      [L,H] fp32: rows [lo, hi) receive the attention output of the
 *            region's queries (q = bf16(x Wq^T)) over all L cached positions,
 *            per head softmax(q k^T / sqrt(d_head)) v; other rows untouched
 *   lo_hi    optional HOST int32[2] receiving the region.
 * The projections and the attention both run on this library's tcgen05
 * kernels.  Errors: ARG (null / bad block), SHAPE (alignment).             */
typedef struct dinfer_kv dinfer_kv;
typedef struct {
  int32_t L, H, d_head;
  int32_t prefix_look, after_look, warmup_times;
} dinfer_kv_shape;
dinfer_status dinfer_kv_create(const dinfer_kv_shape* shape, void* stream, dinfer_kv** out);
void dinfer_kv_destroy(dinfer_kv* kv);
/* host helper: the refresh region [lo, hi) (returns hi - lo, -1 on null args) */
int32_t dinfer_kv_region(const dinfer_kv_shape* shape, int32_t start, int32_t end, int32_t t, int32_t full,
                         int32_t* lo, int32_t* hi);
dinfer_status dinfer_kv_step(dinfer_kv* kv, const uint16_t* X, const uint16_t* Wq, const uint16_t* Wk,
                             const uint16_t* Wv, uint16_t* Kc, uint16_t* Vc, int32_t start, int32_t end,
                             int32_t t, int32_t full, float* out, int32_t* lo_hi);

/* Synchronise the ctx stream and report asynchronous errors (CUDA, NCCL,
 * sticky device-checked preconditions); clears the sticky device flag.      */
dinfer_status dinfer_sync(dinfer_ctx* ctx);
const char* dinfer_strerror(dinfer_status s);
/* Detail of the most recent CUDA/NCCL failure on the calling thread
 * ("<call>: <error string>"), or "" -- diagnostics only.                    */
const char* dinfer_last_error(void);

/* Instrumentation.  dinfer_set_timing(ctx, 1) brackets every kernel / the
 * collective of subsequent steps with CUDA events on the ctx stream;
 * dinfer_get_timing fills up to n floats with the last step's per-phase
 * milliseconds in the order [K1 vocab_proj (or K1b, or K12), K2 smooth_mix,
 * record finalize (K1 paths, sharded / split-phase), C1 allgather, K34
 * select_commit + smooth_finalize, unused] (0 if not run); it
 * synchronises the stream.  dinfer_launches_per_step: kernels the library
 * launches for one dinfer_step with these params (collectives excluded).    */
dinfer_status dinfer_set_timing(dinfer_ctx* ctx, int32_t enable);
dinfer_status dinfer_get_timing(dinfer_ctx* ctx, float* ms, int32_t n);
int32_t dinfer_launches_per_step(const dinfer_ctx* ctx, const dinfer_params* params);

/* Per-CTA kernel timelines (diagnostics).  Only when the process sets
 * DINFER_TRACE=1 before dinfer_create: K1 then K2 CTAs, 5 words each: 4
 * %globaltimer nanosecond stamps (start, first operand stage ready, main loop
 * done, exit) and the SM id, of the most recent step.  Returns the number of words (out == NULL:
 * the number available), 0 if tracing is off.                               */
int32_t dinfer_get_trace(dinfer_ctx* ctx, uint64_t* out, int32_t n);

/* Geometry actually chosen (for reports): grid sizes and pipeline depth.    */
typedef struct {
  int32_t k1_grid, k1_stages, k1_h_resident, k1_smem;
  int32_t k2_grid, k2_hw, k2_groups, k2_stages, k2_smem;
  int32_t num_sms;
  int32_t fused;       /* 1: smoothing steps run K1+K2 as one kernel (K12); its
                          E phase is described by k2_hw / k2_groups / k2_stages */
  int32_t fused_smem;
} dinfer_geometry;
dinfer_status dinfer_get_geometry(const dinfer_ctx* ctx, dinfer_geometry* out);

#ifdef __cplusplus
}
#endif
#endif /* DINFER_H */
