// Device-resident blockwise generation loop:
// Algorithm 1's outer `while` over blocks and inner `while any(undecided)`
// as ONE CUDA graph with a conditional WHILE node, so the
// host never synchronises inside a generation ("without
// control-flow operations ... data transfer from PyTorch tensors to Python
// code is eliminated").  Per iteration the body runs
//     model stand-in (hidden of iteration n)  ->  dinfer_step (K1, K2, K34)
//     ->  gen_control (schedules, block bookkeeping, EOS early termination,
//                      loop condition)
// gen_control / gen_init are single-CTA bookkeeping kernels; all per-step
// arithmetic stays in the step kernels.  Readings c11, c12, c21-c23
// (DESIGN.md): schedules restart per block, tau_t drives tau (threshold) or
// theta_hi (hierarchical); blocks left to right in lockstep over the B rows;
// a row whose completed block holds eos_id is finished and its later blocks
// are EOS-filled; the loop halts when every row is finished.
#include "common.cuh"
#include "kernels.h"

namespace dinfer {
namespace {

constexpr int kGenThreads = 1024;

DI float tau_sched(const GenArgs& a, int t) {  // P:285, reading c11 (linear decay)
  if (a.tau_decay <= 0) return a.tau_target;
  const float frac = static_cast<float>(min(t, a.tau_decay)) / static_cast<float>(a.tau_decay);
  return 1.0f - (1.0f - a.tau_target) * frac;
}
DI float alpha_sched(const GenArgs& a, int t) {
  return fminf(a.a_init + a.a_growth * static_cast<float>(t), a.a_preset);
}

// Step parameters of block-local iteration t -> pdev (read by K34).
DI void write_params(const GenArgs& a, int t) {
  if (threadIdx.x != 0) return;
  for (int j = 0; j < 8; ++j) a.pdev[j] = a.base[j];
  const float thr = tau_sched(a, t);
  if (a.decoder == 0) a.pdev[0] = thr;  // tau
  else a.pdev[1] = thr;                 // theta_hi (theta_lo fixed)
  if (a.use_smooth) a.pdev[6] = alpha_sched(a, t);
}

// Load block st[0] of X into the block-local state (EOS fill for finished
// rows, credit reset P:327, t = 0).  Returns (CTA-uniform) whether any
// position is undecided.
DI int load_block(const GenArgs& a, int* s_any) {
  const int blk = a.st[0];
  const int lo = a.P + blk * a.S;
  if (threadIdx.x == 0) *s_any = 0;
  __syncthreads();
  const int M = a.B * a.S;
  int any = 0;
  for (int b = 0; b < a.B; ++b) {
    const int done = a.st[4 + b];
    for (int s = threadIdx.x; s < a.S; s += blockDim.x) {
      int tok = a.X[static_cast<long>(b) * a.L + lo + s];
      if (done && tok == a.mask_id) tok = a.eos_id;  // finished row: EOS fill (c22)
      a.tokens[b * a.S + s] = tok;
      const int und = tok == a.mask_id;
      a.mask[b * a.S + s] = static_cast<uint8_t>(und);
      any |= und;
    }
  }
  if (a.use_credit) {
    for (int j = threadIdx.x; j < M * a.K; j += blockDim.x) {
      a.cids[j] = -1;
      a.cval[j] = 0.f;
    }
  }
  if (any) atomicOr(s_any, 1);
  __syncthreads();
  return *s_any;
}

DI void write_back(const GenArgs& a) {
  const int lo = a.P + a.st[0] * a.S;
  for (int b = 0; b < a.B; ++b)
    for (int s = threadIdx.x; s < a.S; s += blockDim.x) a.X[static_cast<long>(b) * a.L + lo + s] = a.tokens[b * a.S + s];
}

// Final outputs: T_b (tokens before the first EOS, c23), F, truncated.
DI void finish(const GenArgs& a, int* s_first) {
  for (int b = threadIdx.x; b < a.B; b += blockDim.x) s_first[b] = a.L - a.P;
  __syncthreads();
  for (int b = 0; b < a.B; ++b)
    for (int p = threadIdx.x; p < a.L - a.P; p += blockDim.x)
      if (a.X[static_cast<long>(b) * a.L + a.P + p] == a.eos_id) atomicMin(&s_first[b], p);
  __syncthreads();
  for (int b = threadIdx.x; b < a.B; b += blockDim.x) a.out[b] = s_first[b];
  if (threadIdx.x == 0) {
    a.out[a.B] = a.st[2];
    a.out[a.B + 1] = a.st[3];
  }
}

// The block in st[0] is complete (or about to be skipped): write it back,
// apply early termination, advance to the next block holding an undecided
// position.  Returns whether the loop continues.
DI int advance(const GenArgs& a, bool completed, int* s_flag) {
  for (;;) {
    if (completed) {
      write_back(a);
      if (a.early) {
        // row done <=> its completed block holds eos_id (c22)
        for (int b = 0; b < a.B; ++b)
          for (int s = threadIdx.x; s < a.S; s += blockDim.x)
            if (a.tokens[b * a.S + s] == a.eos_id) a.st[4 + b] = 1;  // benign same-value race
        __syncthreads();
        if (threadIdx.x == 0) {
          int all = 1;
          for (int b = 0; b < a.B; ++b) all &= a.st[4 + b];
          *s_flag = all;
        }
        __syncthreads();
        if (*s_flag) {  // every row finished: fill the remaining blocks, halt
          const int hi = a.P + (a.st[0] + 1) * a.S;
          for (int b = 0; b < a.B; ++b)
            for (int p = hi + threadIdx.x; p < a.L; p += blockDim.x) {
              const long idx = static_cast<long>(b) * a.L + p;
              if (a.X[idx] == a.mask_id) a.X[idx] = a.eos_id;
            }
          __syncthreads();
          return 0;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) a.st[0] += 1;
      __syncthreads();
    }
    if (a.st[0] >= a.nblocks) return 0;
    if (threadIdx.x == 0) a.st[1] = 0;
    if (load_block(a, s_flag)) return 1;
    completed = true;  // nothing undecided in this block: settle it and move on
  }
}

__global__ void __launch_bounds__(kGenThreads) gen_init_kernel(const GenArgs a, cudaGraphConditionalHandle h) {
  __shared__ int s_flag;
  extern __shared__ int s_first[];
  if (threadIdx.x == 0) {
    a.st[0] = 0;  // block
    a.st[1] = 0;  // t (block-local iteration)
    a.st[2] = 0;  // F (forwards)
    a.st[3] = 0;  // truncated
  }
  for (int b = threadIdx.x; b < a.B; b += blockDim.x) a.st[4 + b] = 0;
  __syncthreads();
  int go = advance(a, false, &s_flag);
  if (go && a.max_forwards <= 0) {
    write_back(a);
    if (threadIdx.x == 0) a.st[3] = 1;
    go = 0;
  }
  __syncthreads();
  if (go) write_params(a, 0);
  else finish(a, s_first);
  if (threadIdx.x == 0) cudaGraphSetConditional(h, go ? 1u : 0u);
}

__global__ void __launch_bounds__(kGenThreads) gen_control_kernel(const GenArgs a, cudaGraphConditionalHandle h) {
  __shared__ int s_flag;
  extern __shared__ int s_first[];
  // launched with PDL behind K34: resident while K34 runs, proceeds the
  // moment K34's commit is complete (no launch gap in the loop body)
  grid_dep_wait();
  if (threadIdx.x == 0) {
    a.st[2] += 1;  // F
    a.st[1] += 1;  // t
    s_flag = 0;
  }
  __syncthreads();
  int any = 0;
  for (int i = threadIdx.x; i < a.B * a.S; i += blockDim.x) any |= a.mask[i];
  if (any) atomicOr(&s_flag, 1);
  __syncthreads();
  int go = s_flag ? 1 : advance(a, true, &s_flag);
  __syncthreads();
  if (go && a.st[2] >= a.max_forwards) {  // safety bound: stop with the block written back
    write_back(a);
    __syncthreads();
    if (threadIdx.x == 0) a.st[3] = 1;
    go = 0;
  }
  __syncthreads();
  if (go) write_params(a, a.st[1]);
  else finish(a, s_first);
  if (threadIdx.x == 0) cudaGraphSetConditional(h, go ? 1u : 0u);
}

// Model stand-in: hidden of global iteration n = st[2] (clamped to the
// supplied trajectory) into the step's hidden buffer.
__global__ void gen_hidden_kernel(const GenArgs a) {
  // the step's first kernel (launched with PDL) may start now: it prefetches
  // W (which does not depend on this copy) and waits for the copy before the
  // hidden loads
  grid_dep_launch_dependents();
  const long n = min(static_cast<long>(a.st[2]), a.hsrc_iters - 1);
  const uint4* src = reinterpret_cast<const uint4*>(a.hsrc + n * a.MH);
  uint4* dst = reinterpret_cast<uint4*>(a.hbuf);
  const long nv = a.MH / 8;
  for (long j = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; j < nv; j += gridDim.x * blockDim.x)
    dst[j] = src[j];
}

// Block start (Alg. 1 NextBlock; credit reset P:327): every
// position of the block masked, credit slots empty.  Triggers its dependents
// first, so the next step's kernel (PDL) can start streaming W underneath.
__global__ void block_reset_kernel(uint8_t* mask, int32_t* tokens, int32_t* cids, float* cval, int M, int K,
                                   int mask_id) {
  grid_dep_launch_dependents();
  grid_dep_wait();  // the previous step's commit is complete
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = tid; i < M; i += nt) {
    mask[i] = 1;
    tokens[i] = mask_id;
  }
  if (cids != nullptr)
    for (int i = tid; i < M * K; i += nt) {
      cids[i] = -1;
      cval[i] = 0.f;
    }
}

}  // namespace

cudaError_t launch_block_reset(uint8_t* mask, int32_t* tokens, int32_t* cids, float* cval, int M, int K, int mask_id,
                               cudaStream_t st, bool pdl) {
  return launch_ex(block_reset_kernel, dim3(1), dim3(1024), 0, st, pdl, mask, tokens, cids, cval, M, K, mask_id);
}

cudaError_t launch_gen_init(const GenArgs& a, cudaGraphConditionalHandle h, cudaStream_t st) {
  gen_init_kernel<<<1, kGenThreads, sizeof(int) * a.B, st>>>(a, h);
  return cudaGetLastError();
}
cudaError_t launch_gen_control(const GenArgs& a, cudaGraphConditionalHandle h, cudaStream_t st, bool pdl) {
  return launch_ex(gen_control_kernel, dim3(1), dim3(kGenThreads), sizeof(int) * a.B, st, pdl, a, h);
}
cudaError_t launch_gen_hidden(const GenArgs& a, int grid, cudaStream_t st) {
  gen_hidden_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace dinfer
