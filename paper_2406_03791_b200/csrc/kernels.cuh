// kernels.cuh — the decoder's sm_100a kernels (graph path).
//
//   (K1, the tcgen05 3xTF32 encoder projection, lives in encproj_tc.cuh)
//   prologue_kernel       K0 state / emission / loop-flag initialisation
//   pred_layer_kernel     K2 one prediction-network layer: gate GEMV fused with
//                         the tanh / LSTM cell and the predicated state commit
//   pred_proj_kernel      gp = h_top @ pred_proj (cached per accepted label)
//   joint_kernel          K3 joint step: relu(fp+gp) @ out_proj(||dur_proj),
//                         per-chunk log-sum-exp + argmax, last-CTA decision
//                         (blank mask / label-loop cursor rules, hypothesis +
//                         timestamp append, loop flag, cudaGraphSetConditional)
//   frame_tail_kernel     frame-sync outer-loop tail (t += 1, next frame init)
//
// Per-output arithmetic is fp32 with FFMA; reductions run in a fixed order so
// every launch is deterministic.  Reference semantics cited per function.
#pragma once

#include "common.cuh"

namespace rnntg {

// -------------------------------------------------------------------------
// Step GEMV building block.
// One warp accumulates a 32-row x 16-col tile over its k-slice [k0, k0+kw):
//   lane = (rg = lane>>2 : rows rg, rg+8, rg+16, rg+24) x (cg = lane&3 : cols 4cg..4cg+3)
// A rows come from shared memory (row stride KS, KS % 32 == 4 so the 8 row
// groups hit 8 distinct bank quads: one wavefront per LDS.128, broadcast over
// cg).  W is stored tiled ([tile][K][16], contiguous per warp slice) and is
// streamed through the warp's own shared-memory slot by bulk copies of WCH
// k-rows (4 KB): bulk copies issued by one warp serialise, so every warp
// issues its own (scripts/microbench3.cu), and the first chunk is requested
// before griddepcontrol.wait because weights never depend on the previous
// kernel.  kw must be a multiple of 8.
// -------------------------------------------------------------------------
constexpr int WCH = 64;  // W k-rows per bulk copy (64 x 16 floats = 4 KB)

__device__ __forceinline__ void w_chunk_issue(const float* Wslice, int kc, int nk, float* wslot,
                                              uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_arrive_expect_tx(bar, (uint32_t)(nk * CT * sizeof(float)));
  bulk_g2s(wslot, Wslice + (size_t)kc * CT, (uint32_t)(nk * CT * sizeof(float)), bar);
}

__device__ __forceinline__ void warp_gemv_32x16(const float* __restrict__ As, int KS,
                                                const float* __restrict__ Wslice, int k0, int kw,
                                                float* wslot, uint64_t* wbar, bool first_issued,
                                                float (&acc)[4][4]) {
  const int lane = threadIdx.x & 31, rg = lane >> 2, cg = lane & 3;
  const float* ap = As + rg * KS + k0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
  uint32_t ph = 0;
  for (int kc = 0; kc < kw; kc += WCH) {
    const int nk = kw - kc < WCH ? kw - kc : WCH;
    if (lane == 0 && !(kc == 0 && first_issued)) w_chunk_issue(Wslice, kc, nk, wslot, wbar);
    mbar_wait(wbar, ph);
    ph ^= 1u;
    const float* wr = wslot + 4 * cg;
#pragma unroll 2
    for (int k = 0; k < nk; k += 4) {
      const float4 w0 = lds4(wr + (k + 0) * CT), w1 = lds4(wr + (k + 1) * CT),
                   w2 = lds4(wr + (k + 2) * CT), w3 = lds4(wr + (k + 3) * CT);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 a = lds4(ap + i * 8 * KS + kc + k);
        acc[i][0] = fmaf(a.x, w0.x, acc[i][0]);
        acc[i][1] = fmaf(a.x, w0.y, acc[i][1]);
        acc[i][2] = fmaf(a.x, w0.z, acc[i][2]);
        acc[i][3] = fmaf(a.x, w0.w, acc[i][3]);
        acc[i][0] = fmaf(a.y, w1.x, acc[i][0]);
        acc[i][1] = fmaf(a.y, w1.y, acc[i][1]);
        acc[i][2] = fmaf(a.y, w1.z, acc[i][2]);
        acc[i][3] = fmaf(a.y, w1.w, acc[i][3]);
        acc[i][0] = fmaf(a.z, w2.x, acc[i][0]);
        acc[i][1] = fmaf(a.z, w2.y, acc[i][1]);
        acc[i][2] = fmaf(a.z, w2.z, acc[i][2]);
        acc[i][3] = fmaf(a.z, w2.w, acc[i][3]);
        acc[i][0] = fmaf(a.w, w3.x, acc[i][0]);
        acc[i][1] = fmaf(a.w, w3.y, acc[i][1]);
        acc[i][2] = fmaf(a.w, w3.z, acc[i][2]);
        acc[i][3] = fmaf(a.w, w3.w, acc[i][3]);
      }
    }
    __syncwarp();
  }
}

// Store a warp's partial tile into red[warp][32][16].
__device__ __forceinline__ void store_partial(float* red, const float (&acc)[4][4]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, rg = lane >> 2, cg = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float4 v = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    *reinterpret_cast<float4*>(red + ((warp * RB) + rg + 8 * i) * CT + 4 * cg) = v;
  }
}

// Sum of the NW warp partials for (row r, col c), fixed warp order.
__device__ __forceinline__ float reduce_partial(const float* red, int r, int c) {
  float s = red[r * CT + c];
#pragma unroll
  for (int w = 1; w < NW; ++w) s += red[(w * RB + r) * CT + c];
  return s;
}

// Shared-memory carve-up of the step kernels:
// [NW A-mbarriers][NW W-mbarriers][flag][As 32 x KS][red][NW W slots].
struct StepSmem {
  uint64_t* bars;
  uint64_t* wbars;
  float* As;
  float* red;
  float* wslots;
  int* flag;
};
__device__ __forceinline__ StepSmem carve(void* base, int KS) {
  StepSmem s;
  s.bars = reinterpret_cast<uint64_t*>(base);
  s.wbars = s.bars + NW;
  s.flag = reinterpret_cast<int*>(s.wbars + NW);
  s.As = reinterpret_cast<float*>(reinterpret_cast<char*>(base) + 256);
  s.red = s.As + RB * KS;
  s.wslots = s.red + NW * RB * CT;
  return s;
}
__host__ __device__ inline size_t step_smem_bytes(int K) {
  return 256 + sizeof(float) * ((size_t)RB * (K + 4) + (size_t)NW * RB * CT + (size_t)NW * WCH * CT);
}

// Per-warp W slot and the first-chunk prefetch (issued before the PDL wait).
__device__ __forceinline__ float* warp_wslot(const StepSmem& sm) {
  return sm.wslots + (threadIdx.x >> 5) * WCH * CT;
}
__device__ __forceinline__ void init_step_barriers(const StepSmem& sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    mbar_init(&sm.bars[warp], 1);
    mbar_init(&sm.wbars[warp], 1);
  }
  fence_mbar_init();
  __syncwarp();
}
__device__ __forceinline__ void prefetch_w(const StepSmem& sm, const float* Wslice, int kw) {
  if ((threadIdx.x & 31) == 0)
    w_chunk_issue(Wslice, 0, kw < WCH ? kw : WCH, warp_wslot(sm), &sm.wbars[threadIdx.x >> 5]);
}

// Stage this warp's k-slice of 32 activation rows with the bulk-copy (TMA)
// engine.  Sources: k < seg_k from src0, else from src1 (both [rows][ld]).
__device__ __forceinline__ void stage_rows_bulk(const StepSmem& sm, int KS, int row0,
                                                const float* src0, const float* src1, int seg_k,
                                                int ld, int k0, int kw) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* src = k0 < seg_k ? src0 : src1;
  const int koff = k0 < seg_k ? k0 : k0 - seg_k;
  // Rows are not contiguous in global memory, so a per-row bulk copy would
  // issue 32 serialised copies per warp; 16-byte cp.async from every lane
  // keeps all of them in flight instead.
  (void)warp;
  const int q4 = kw / 4;
  for (int p = lane; p < RB * q4; p += 32) {
    const int r = p / q4, q = p % q4;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm.As + r * KS + k0 + 4 * q)),
                 "l"(src + (size_t)(row0 + r) * ld + koff + 4 * q)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncwarp();
}

// -------------------------------------------------------------------------
// Exact table of the layer-0 input contribution: table0[v, col] =
// sum_e embedding[v, e] * W_ih0[e, col], sequential e with separate rounding
// per multiply and add -- bit-identical to the reference's pred.matmul_ih
// (model.cpp:338-342, tensor.cpp:249-257) for every label, computed once.
// -------------------------------------------------------------------------
__global__ void table0_kernel(const float* __restrict__ emb, const float* __restrict__ wih,
                              float* __restrict__ table, int V1, int E, int ncols_in,
                              int G, int H, int Hp) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;  // reference column g*H + u
  const int v = blockIdx.y;
  if (col >= ncols_in || v >= V1) return;
  float acc = 0.0f;
  for (int e = 0; e < E; ++e)
    acc = __fadd_rn(acc, __fmul_rn(emb[(size_t)v * E + e], wih[(size_t)e * ncols_in + col]));
  const int g = col / H, u = col % H;
  table[(size_t)v * (G * Hp) + u * G + g] = acc;
}

// -------------------------------------------------------------------------
// K0 prologue: launch_fs_prologue / launch_ll_prologue (decoders.cpp:216-233,
// 414-430): zero the prediction state, counts, last_label = blank, loop
// scalars; frame-sync: blank mask for frame 0; label-loop: t = u = 0,
// active = t < out_len.  Every row is marked `accept` so the following
// prediction step computes P0 = pred(blank, 0) for all rows.
// -------------------------------------------------------------------------
__global__ void prologue_kernel(DevModel M, DevState S) {
  // zero state (both parities) with a grid-stride loop
  const size_t nstate = (size_t)S.Bp * M.Hp;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t nthr = (size_t)gridDim.x * blockDim.x;
  for (int l = 0; l < M.L; ++l)
    for (int p = 0; p < 2; ++p) {
      for (size_t i = tid; i < nstate; i += nthr) {
        S.h[l][p][i] = 0.0f;
        if (S.c[l][p]) S.c[l][p][i] = 0.0f;
      }
    }
  for (size_t i = tid; i < (size_t)S.Bp * M.Jp; i += nthr) S.gp[i] = 0.0f;
  if (blockIdx.x != 0) return;
  __shared__ int smax;
  __shared__ int sany;
  if (threadIdx.x == 0) {
    smax = 0;
    sany = 0;
  }
  __syncthreads();
  const int blank = M.V1 - 1;
  for (int b = threadIdx.x; b < S.Bp; b += blockDim.x) {
    const int len = b < S.B ? S.out_len[b] : 0;
    const int live = b < S.B;
    S.last_label[b] = blank;
    S.accept[b] = live;
    S.counts[b] = 0;
    S.t_row[b] = 0;
    S.u_row[b] = 0;
    S.done[b] = live ? (0 >= len) : 1;
    const int act = live && (0 < len);
    S.active[b] = act;
    S.need[b] = act;
    if (live) atomicMax(&smax, len);
    if (act) sany = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Ctrl* c = S.ctrl;
    c->t = 0;
    c->sym = 0;
    c->max_len = smax;
    c->par = 0;
    c->err = 0;
    c->abort = 0;
    c->any = sany;
    for (int i = 0; i < MAXRB; ++i) c->ctr_joint_rb[i] = 0;
    c->ctr_joint_all = 0;
    c->ctr_pp = 0;
    c->joint_evals = 0;
    c->pred_steps = 0;
    c->outer_iters = 0;
    c->iters = 0;
    if (S.use_cond) {
      if (S.algo == ALGO_FS) {
        cudaGraphSetConditional(S.h_outer, smax > 0 ? 1u : 0u);
        cudaGraphSetConditional(S.h_inner, 1u);
      }
      // label-loop conditions are set by the prologue's pred_proj tail
    }
  }
}

// -------------------------------------------------------------------------
// K2: one prediction-network layer for every row of a 32-row block and one
// 16-column tile of gate columns (4 LSTM units or 16 tanh units).
//   tanh (model.cpp:163-176, 39-51):  h' = tanh((ih + hh) + bias)
//   LSTM:          gates = (ih + hh) + b ; i,f,g,o ;
//                                     c' = f c + i g ; h' = o tanh(c')
// Layer 0's ih comes from the exact table0[last_label]; layers > 0 fold ih
// into the GEMV over [h_{l-1}' | h_l].  Rows that did not accept a label copy
// their old state (where_select_rows semantics, decoders.cpp:292-295).
// -------------------------------------------------------------------------
template <int CELL>
__global__ void __launch_bounds__(NT) pred_layer_kernel(DevModel M, DevState S, int l) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int K = l == 0 ? M.Hp : 2 * M.Hp;
  const int KS = K + 4;
  StepSmem sm = carve(smem_raw, KS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, rb = blockIdx.y, row0 = rb * RB, col0 = tile * CT;
  const int kw = K / NW, k0 = warp * kw;
  const float* wslice = M.w[l] + ((size_t)tile * K + k0) * CT;  // tiled [tile][K][16]
  init_step_barriers(sm);
  prefetch_w(sm, wslice, kw);
  pdl_trigger();
  pdl_wait();
  const int par = ld_volatile(&S.ctrl->par);
  const int cur = par, nxt = par ^ 1;
  if (l == 0)
    stage_rows_bulk(sm, KS, row0, S.h[0][cur], S.h[0][cur], K, M.Hp, k0, kw);
  else
    stage_rows_bulk(sm, KS, row0, S.h[l - 1][nxt], S.h[l][cur], M.Hp, M.Hp, k0, kw);
  float acc[4][4];
  warp_gemv_32x16(sm.As, KS, wslice, k0, kw, warp_wslot(sm), &sm.wbars[warp], true, acc);
  store_partial(sm.red, acc);
  __syncthreads();
  const float* bias = M.bias[l];
  if (CELL == 1) {
    // 4 units x 32 rows; thread -> (row, unit)
    if (threadIdx.x < RB * 4) {
      const int r = threadIdx.x >> 2, uu = threadIdx.x & 3;
      const int b = row0 + r;
      const int u = tile * 4 + uu;
      if (b < S.B) {
        float gt[4];
        const int lab = S.last_label[b];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int col = uu * 4 + g;
          float hh = reduce_partial(sm.red, r, col);
          float pre = l == 0 ? M.table0[(size_t)lab * M.GH + col0 + col] + hh : hh;
          gt[g] = pre + bias[col0 + col];
        }
        const size_t idx = (size_t)b * M.Hp + u;
        const float c_old = S.c[l][cur][idx];
        float hn, cn;
        if (S.accept[b]) {
          const float i_ = sigmoid_f(gt[0]), f_ = sigmoid_f(gt[1]);
          const float g_ = tanhf(gt[2]), o_ = sigmoid_f(gt[3]);
          cn = f_ * c_old + i_ * g_;
          hn = o_ * tanhf(cn);
        } else {
          cn = c_old;
          hn = S.h[l][cur][idx];
        }
        S.c[l][nxt][idx] = cn;
        S.h[l][nxt][idx] = hn;
      }
    }
  } else {
    for (int o = threadIdx.x; o < RB * CT; o += NT) {
      const int r = o / CT, col = o % CT;
      const int b = row0 + r;
      if (b >= S.B) continue;
      const int u = col0 + col;
      const size_t idx = (size_t)b * M.Hp + u;
      float hn;
      if (S.accept[b]) {
        const float hh = reduce_partial(sm.red, r, col);
        const int lab = S.last_label[b];
        hn = tanhf((M.table0[(size_t)lab * M.GH + u] + hh) + bias[u]);
      } else {
        hn = S.h[0][cur][idx];
      }
      S.h[0][nxt][idx] = hn;
    }
  }
}

// -------------------------------------------------------------------------
// Label-loop bookkeeping after a prediction step (end of launch_ll_body,
// decoders.cpp:485-512 + active_update 402-412): every active row needs a
// decision in the next round; loop flags for the nested WHILE nodes.
// -------------------------------------------------------------------------
__device__ void ll_round_tail(const DevModel& M, const DevState& S) {
  __shared__ int s_any;
  if (threadIdx.x == 0) s_any = 0;
  __syncthreads();
  int any = 0;
  for (int b = threadIdx.x; b < S.B; b += blockDim.x) {
    const int act = S.active[b];
    S.need[b] = act;
    S.accept[b] = 0;
    any |= act;
  }
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) {
    Ctrl* c = S.ctrl;
    const int go = any && !c->abort;
    c->any = go;
    c->outer_iters += 1;
    if (S.use_cond) {
      cudaGraphSetConditional(S.h_inner, go ? 1u : 0u);
      cudaGraphSetConditional(S.h_outer, go ? 1u : 0u);
    }
  }
}

// -------------------------------------------------------------------------
// gp = h_top' @ pred_proj for accepted rows (joint.pred_proj, model.cpp:370-374,
// cached per prediction state -- bit-neutral).  The last
// CTA flips the state parity and runs the label-loop round tail.
// -------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) pred_proj_kernel(DevModel M, DevState S) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int K = M.Hp, KS = K + 4;
  StepSmem sm = carve(smem_raw, KS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, rb = blockIdx.y, row0 = rb * RB, col0 = tile * CT;
  const int kw = K / NW, k0 = warp * kw;
  const float* wslice = M.pred_proj + ((size_t)tile * K + k0) * CT;  // tiled [tile][Hp][16]
  (void)lane;
  init_step_barriers(sm);
  prefetch_w(sm, wslice, kw);
  pdl_trigger();
  pdl_wait();
  const int nxt = ld_volatile(&S.ctrl->par) ^ 1;
  const float* htop = S.h[M.L - 1][nxt];
  stage_rows_bulk(sm, KS, row0, htop, htop, K, M.Hp, k0, kw);
  float acc[4][4];
  warp_gemv_32x16(sm.As, KS, wslice, k0, kw, warp_wslot(sm), &sm.wbars[warp], true, acc);
  store_partial(sm.red, acc);
  __syncthreads();
  for (int o = threadIdx.x; o < RB * CT; o += NT) {
    const int r = o / CT, col = o % CT, b = row0 + r;
    if (b < S.B && S.accept[b]) S.gp[(size_t)b * M.Jp + col0 + col] = reduce_partial(sm.red, r, col);
  }
  // last CTA of the grid: parity flip + loop bookkeeping
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned total = gridDim.x * gridDim.y;
    const unsigned prev = atomicAdd(&S.ctrl->ctr_pp, 1u);
    *sm.flag = (prev == total - 1);
  }
  __syncthreads();
  if (!*sm.flag) return;
  __threadfence();
  if (threadIdx.x == 0) {
    S.ctrl->ctr_pp = 0;
    S.ctrl->par ^= 1;
    S.ctrl->pred_steps += 1;
  }
  if (S.algo != ALGO_FS) ll_round_tail(M, S);
}

// -------------------------------------------------------------------------
// Scripted model prediction step (ScriptedModel::run_prediction,
// model.cpp:563-572): the state is the running emission count,
// hidden' = hidden + 1 for the rows that accepted a label (where_select_rows,
// decoders.cpp:292-295); the "projection" gp[b][0] is the committed state the
// joint reads as g.  One CTA; the tail is pred_proj_kernel's (parity flip,
// pred_steps, label-loop round bookkeeping).
// -------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) scripted_pred_kernel(DevModel M, DevState S) {
  pdl_trigger();
  pdl_wait();
  const int par = ld_volatile(&S.ctrl->par), cur = par, nxt = par ^ 1;
  for (int b = threadIdx.x; b < S.B; b += blockDim.x) {
    const size_t idx = (size_t)b * M.Hp;
    const float h = S.h[0][cur][idx];
    if (S.accept[b]) {
      S.h[0][nxt][idx] = h + 1.0f;
      S.gp[(size_t)b * M.Jp] = h + 1.0f;
    } else {
      S.h[0][nxt][idx] = h;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    S.ctrl->ctr_pp = 0;
    S.ctrl->par ^= 1;
    S.ctrl->pred_steps += 1;
  }
  if (S.algo != ALGO_FS) ll_round_tail(M, S);
}

// Scripted model joint logit (ScriptedModel::run_joint / run_joint_tdt,
// model.cpp:574-615): 10 on the planted label (or duration class) of the
// decision at (b, t, u), 0 elsewhere; u = emissions so far - emissions on
// arrival at frame t (frame-sync arrivals for run_joint, duration-schedule
// arrivals for run_joint_tdt).  col: vocab column, or duration class index
// when dur.
__device__ __forceinline__ float scripted_logit(const DevModel& M, const DevState& S, int b, int t, int col,
                                                bool dur) {
  const int blank = M.V1 - 1;
  const int emitted = (int)S.gp[(size_t)b * M.Jp] - 1;
  const bool in = b < M.s_B && t < M.s_T;
  int u;
  if (S.algo == ALGO_TDT) {
    const int arr = in ? M.s_darr[(size_t)b * M.s_T + t] : -1;
    u = arr < 0 ? -1 : emitted - arr;
  } else {
    const int tt = t < 0 ? 0 : (t > M.s_T ? M.s_T : t);
    u = emitted - (b < M.s_B ? M.s_fsarr[(size_t)b * (M.s_T + 1) + tt] : 0);
  }
  if (!dur) {
    const int lab = (in && u >= 0 && u < M.s_U) ? M.s_lab[((size_t)b * M.s_T + t) * M.s_U + u] : blank;
    return col == lab ? 10.0f : 0.0f;
  }
  // duration_at(b, t, u < 0 ? 1 << 20 : u): the entry index is min(u, len)
  int d;
  if (in) {
    const int ui = (u < 0 || u > M.s_U) ? M.s_U : u;
    d = M.s_dval[((size_t)b * M.s_T + t) * (M.s_U + 1) + ui];
  } else {
    d = 1;  // blank outside the table
  }
  int cls = 0;
  for (int i = 0; i < M.D; ++i)
    if (M.durations[i] == d) {
      cls = i;
      break;
    }
  return col == cls ? 10.0f : 0.0f;
}

// -------------------------------------------------------------------------
// Per-row decision of the joint step (lane 0 of the row's warp).
//   frame-sync: launch_fs_inner_body's argmax/blank_update/save_kv/update_*
//               (decoders.cpp:261-307)
//   label-loop / TDT: accept_mask, save_kv, commit_last_label, step_advance,
//               active_update (decoders.cpp:432-512)
// -------------------------------------------------------------------------
__device__ __forceinline__ void append_emission(const DevState& S, int b, int k, int frame,
                                                float v, int dur) {
  const int n = S.counts[b];
  if (n < S.cap) {  // unreachable bound, decoders.cpp:81
    const size_t o = (size_t)b * S.cap + n;
    S.tokens[o] = k;
    S.frames[o] = frame;
    S.scores[o] = v;
    S.durs[o] = dur;
    S.counts[b] = n + 1;
  }
}

__device__ __forceinline__ void decide_row(const DevModel& M, const DevState& S, int b, int k,
                                           float v, int dur_idx) {
  const int blank = M.V1 - 1;
  if (S.algo == ALGO_FS) {
    if (S.done[b]) {
      S.accept[b] = 0;
      return;
    }
    if (k == blank) {
      S.done[b] = 1;
      S.accept[b] = 0;
    } else {
      append_emission(S, b, k, S.ctrl->t, v, 0);
      S.last_label[b] = k;
      S.accept[b] = 1;
    }
    return;
  }
  if (!S.need[b]) return;
  const int len = S.out_len[b];
  int t = S.t_row[b], u = S.u_row[b];
  const bool tdt = S.algo == ALGO_TDT;
  if (k == blank) {
    const int d = tdt ? M.durations[dur_idx] : 1;
    t += d > 1 ? d : 1;
    u = 0;
    const int act = t < len;
    S.active[b] = act;
    S.need[b] = act;
  } else {
    const int d = tdt ? M.durations[dur_idx] : 0;
    append_emission(S, b, k, t, v, d);
    S.last_label[b] = k;
    S.accept[b] = 1;
    u += 1;
    if (d > 0) {
      t += d;
      u = 0;
    } else if (u == S.ms) {
      t += 1;
      u = 0;
    }
    S.active[b] = t < len;
    S.need[b] = 0;
  }
  S.t_row[b] = t;
  S.u_row[b] = u;
}

// -------------------------------------------------------------------------
// K3 joint step.  grid = (NCHT column chunks, row blocks).  Each CTA stages
// trunk = relu(fp[b, t_b] + gp[b]) (joint.combine, model.cpp:375-379) for the
// rows that need a decision, computes its 16 logits per row
// (joint.out_proj / dur_proj, model.cpp:380-384, 401-405), and publishes the
// chunk's (max, sum exp(x - max), best value, best index).  The last CTA of a
// row block merges the chunks in fixed order into lse = m + log(s)
// (log_softmax_into, tensor.cpp:463-480) and the lowest-index argmax
// (argmax_last_into, tensor.cpp:268-312), applies the decision rules and
// appends (token, frame, score, duration); the last row block then sets the
// loop flag with cudaGraphSetConditional.
// -------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) joint_kernel(DevModel M, DevState S) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int K = M.Jp, KS = K + 4;
  StepSmem sm = carve(smem_raw, KS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunk = blockIdx.x, rb = blockIdx.y, row0 = rb * RB, col0 = chunk * CT;
  const bool dur_chunk = chunk >= M.NCH;
  const int kw = K / NW, k0 = warp * kw, kq = kw / 4;
  const float* wslice = M.out_ext + ((size_t)chunk * K + k0) * CT;  // tiled [chunk][Jp][16]
  const bool scripted = M.cell == RNNTG_CELL_SCRIPTED;
  init_step_barriers(sm);
  if (!scripted) prefetch_w(sm, wslice, kw);
  pdl_trigger();
  pdl_wait();
  const bool fs = S.algo == ALGO_FS;
  const int tf = fs ? ld_volatile(&S.ctrl->t) : 0;
  // ---- stage trunk rows (this warp's k-slice) ----
  for (int p = lane; p < RB * kq && !scripted; p += 32) {
    const int r = p / kq, q = p % kq, b = row0 + r;
    const int k = k0 + 4 * q;
    float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    bool live = b < S.B && (fs ? !S.done[b] : S.need[b] != 0);
    if (live) {
      int t = fs ? tf : S.t_row[b];
      t = t < 0 ? 0 : (t > S.T - 1 ? S.T - 1 : t);
      const float4 f = ldg4(S.fp + ((size_t)b * S.T + t) * M.Jp + k);
      const float4 g = *reinterpret_cast<const float4*>(S.gp + (size_t)b * M.Jp + k);
      z.x = fmaxf(f.x + g.x, 0.0f);
      z.y = fmaxf(f.y + g.y, 0.0f);
      z.z = fmaxf(f.z + g.z, 0.0f);
      z.w = fmaxf(f.w + g.w, 0.0f);
    }
    *reinterpret_cast<float4*>(sm.As + r * KS + k) = z;
  }
  __syncwarp();
  if (!scripted) {
    float acc[4][4];
    warp_gemv_32x16(sm.As, KS, wslice, k0, kw, warp_wslot(sm), &sm.wbars[warp], true, acc);
    store_partial(sm.red, acc);
  }
  __syncthreads();
  // ---- per-row chunk statistics: half-warp per row ----
  const int half = lane >> 4, hl = lane & 15;
  const int nvalid = dur_chunk ? M.D : (M.V1 - col0 < CT ? M.V1 - col0 : CT);
  for (int r = warp * 2 + half; r < RB; r += 2 * NW) {
    const int b = row0 + r;
    const bool valid = hl < nvalid;
    float x;
    if (scripted) {
      const int t = fs ? tf : (b < S.B ? S.t_row[b] : 0);
      x = b < S.B ? scripted_logit(M, S, b, t < 0 ? 0 : (t > S.T - 1 ? S.T - 1 : t), dur_chunk ? hl : col0 + hl,
                                   dur_chunk)
                  : 0.0f;
    } else {
      x = reduce_partial(sm.red, r, hl);
    }
    if (S.dbg_logits && b < S.B && valid) S.dbg_logits[(size_t)b * M.NOUT + col0 + hl] = x;
    float m = valid ? x : -INFINITY;
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float e = valid ? expf(x - m) : 0.0f;
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    float bv = valid ? x : -INFINITY;
    int bi = valid ? hl : CT;
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (hl == 0 && b < S.Bp)
      S.part[(size_t)b * M.NCHT + chunk] =
          make_float4(m, e, bv, __int_as_float((dur_chunk ? 0 : col0) + bi));
  }
  // ---- last CTA of this row block decides its rows ----
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&S.ctrl->ctr_joint_rb[rb], 1u);
    *sm.flag = (prev == (unsigned)gridDim.x - 1);
  }
  __syncthreads();
  if (!*sm.flag) return;
  __threadfence();
  for (int r = warp; r < RB; r += NW) {
    const int b = row0 + r;
    if (b >= S.B) continue;
    const bool live = fs ? !S.done[b] : S.need[b] != 0;
    if (!live) {
      if (lane == 0 && fs) S.accept[b] = 0;
      continue;
    }
    float Mx = -INFINITY, Sx = 0.0f, best = -INFINITY;
    int bidx = 0x7fffffff;
    for (int c = lane; c < M.NCH; c += 32) {
      const float4 p = __ldcg(&S.part[(size_t)b * M.NCHT + c]);
      const float nm = fmaxf(Mx, p.x);
      Sx = (Sx == 0.0f ? 0.0f : Sx * expf(Mx - nm)) + p.y * expf(p.x - nm);
      Mx = nm;
      const int pi = __float_as_int(p.w);
      if (p.z > best || (p.z == best && pi < bidx)) {
        best = p.z;
        bidx = pi;
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, Mx, o);
      const float os = __shfl_xor_sync(0xffffffffu, Sx, o);
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      const float nm = fmaxf(Mx, om);
      const float a = Sx == 0.0f ? 0.0f : Sx * expf(Mx - nm);
      const float bb = os == 0.0f ? 0.0f : os * expf(om - nm);
      Sx = a + bb;
      Mx = nm;
      if (ob > best || (ob == best && oi < bidx)) {
        best = ob;
        bidx = oi;
      }
    }
    if (lane == 0) {
      const float lse = Mx + logf(Sx);
      const float v = best - lse;
      int dur_idx = 0;
      float lse_d = 0.0f;
      if (M.D > 0) {
        const float4 pd = __ldcg(&S.part[(size_t)b * M.NCHT + M.NCH]);
        dur_idx = __float_as_int(pd.w);
        lse_d = pd.x + logf(pd.y);
      }
      if (S.dbg_lse) {
        S.dbg_lse[b] = lse;
        S.dbg_lse[S.Bp + b] = lse_d;
      }
      decide_row(M, S, b, bidx, v, dur_idx);
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    S.ctrl->ctr_joint_rb[rb] = 0;
    const unsigned prev = atomicAdd(&S.ctrl->ctr_joint_all, 1u);
    *sm.flag = (prev == (unsigned)gridDim.y - 1);
  }
  __syncthreads();
  if (!*sm.flag) return;
  __threadfence();
  // ---- last row block: loop flag ----
  int any = 0;
  for (int b = threadIdx.x; b < S.B; b += blockDim.x)
    any |= fs ? !ld_volatile(&S.done[b]) : ld_volatile(&S.need[b]);
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) {
    Ctrl* c = S.ctrl;
    c->ctr_joint_all = 0;
    c->joint_evals += 1;
    c->iters += 1;
    int go;
    if (fs) {
      c->sym += 1;
      go = any && c->sym < S.ms;
    } else {
      go = any;
    }
    if (c->iters > S.max_iters) {
      c->err = ERR_RUNAWAY;
      c->abort = 1;
      go = 0;
    }
    c->any = go;
    if (S.use_cond) cudaGraphSetConditional(S.h_inner, go ? 1u : 0u);
  }
}

// -------------------------------------------------------------------------
// Frame-sync outer tail: launch_fs_outer_tail + next launch_fs_frame_head's
// frame_init (decoders.cpp:235-259, 309-313): t += 1; blank_mask = t >=
// out_len; symbols_added = 0; inner flag = 1; outer flag = t < max_out_len.
// -------------------------------------------------------------------------
__global__ void frame_tail_kernel(DevModel M, DevState S) {
  pdl_wait();
  const int t = S.ctrl->t + 1;
  for (int b = threadIdx.x; b < S.B; b += blockDim.x) S.done[b] = t >= S.out_len[b];
  __syncthreads();
  if (threadIdx.x == 0) {
    Ctrl* c = S.ctrl;
    c->t = t;
    c->sym = 0;
    c->outer_iters += 1;
    const int go = t < c->max_len && !c->abort;
    if (S.use_cond) {
      cudaGraphSetConditional(S.h_outer, go ? 1u : 0u);
      cudaGraphSetConditional(S.h_inner, 1u);
    }
  }
}

// Marks every row live for standalone kernel timing (rnntg_time_kernel).
__global__ void timing_prep_kernel(DevState S) {
  for (int b = threadIdx.x; b < S.Bp; b += blockDim.x) {
    const int live = b < S.B;
    S.done[b] = !live;
    S.need[b] = live;
    S.accept[b] = live;
    S.counts[b] = 0;
  }
  if (threadIdx.x == 0) {
    S.ctrl->sym = 0;
    S.ctrl->iters = 0;
    S.ctrl->t = 0;
  }
}

}  // namespace rnntg
