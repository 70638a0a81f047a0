// persistent.cuh — K5: the whole decode loop in ONE cooperative persistent
// kernel (the "persistent-kernel alternative" to the conditional-node graph).
//
// Every CTA (one per SM) keeps its slice of the prediction/joint weights
// resident in shared memory for the entire decode and streams only the
// per-step activations through a TMA bulk-copy ring:
//
//   owned by CTA c        smem (C2: 2x640 LSTM, J=640, V=1025)
//   LSTM units [u0,u1)    W_hh0[Hp][20]  (layer-0 recurrent gates)
//                         W_1 [2Hp][20]  (layer-1 [ih;hh] gates)
//   pred_proj cols        W_pp[Hp][8]
//   joint cols            W_J [Jp][8]    (out_proj || dur_proj columns)
//
// One inner step (frame-sync) or label-loop iteration:
//   J   trunk @ W_J -> per-CTA (max, sumexp, best, idx)       -> grid barrier
//   D   every CTA merges all partials for all rows (redundant,
//       identical): argmax / lse / decision rules; CTA 0 appends
//       the hypothesis; layer-0 cell for own units using the
//       exact table0[label] + precomputed h0 @ W_hh0            -> grid barrier
//   P1  [h0'|h1] @ W_1 -> layer-1 cell for own units; h0' @ W_hh0
//       for the next step                                       -> grid barrier
//   Pp  h1' @ W_pp -> gp (accepted rows) and trunk = relu(fp[t]+gp) -> barrier
// Steps where no row accepted a label skip the prediction phases (the
// trunk is refreshed in D instead), exactly like the reference commits
// prediction state only for accepted rows (decoders.cpp:292-295, 474-482).
//
// All per-row control state (labels, cursors, masks) is replicated in every
// CTA's shared memory and updated identically, so only activations, joint
// partials and emissions touch global memory.
#pragma once

#include "common.cuh"
#include "kernels.cuh"

namespace rnntg {
namespace pk {

constexpr int C1 = 20;          // gate columns per CTA (5 LSTM units / 20 tanh units)
constexpr int C2 = 8;           // pred_proj / joint columns per CTA
constexpr int UMAX_LSTM = 5;
constexpr int UMAX_TANH = 20;
constexpr int NCW = 8;          // warps; each streams its own k-slice
constexpr int NTH = NCW * 32;
constexpr int MAXB = 256;       // rows per decoder in the persistent path
constexpr int MAX_NS = 4;       // slot sizes tried: ns * 8 features (32, 24, 16)
constexpr int RED_FLOATS = NCW * RB * C1;

struct PParams {
  int G;            // CTAs
  int B, nrb, T, ms, cap, algo, L, cell;
  int H, Hp, J, Jp, V1, D, NJ;   // NJ = V1 + D joint columns
  int ns;           // per-warp slot = ns * 8 features x 32 rows (bulk-copy granule)
  int own_smem;     // 1: hh0own / cown / gpown live in shared memory
  int dc0, dc1;     // CTAs owning duration columns: [dc0, dc1)
  long long max_iters;
  int durations[MAXD];
  const float* wpack;   // [G][wfloats] packed per-CTA weights
  int wfloats;          // floats per CTA in wpack
  int off_hh0, off_w1, off_pp, off_j;  // float offsets inside a CTA's pack
  const float* bias;    // [G][2][C1] per-CTA bias of owned gate columns (layer 0, 1)
  const float* table0;  // [V1][GH] (graph-path layout, col = u*G + g)
  int GH, Gg;           // GH = Gg*Hp
  const float* fp;      // [B*T][Jp]
  const int* out_len;
  float* h0;            // [nrb][Hp][32] k-major, row index swizzled
  float* h1[2];         // same, ping-pong
  float* trunk;         // [nrb][Jp][32]
  float* hh0own;        // [G][B][C1]
  float* cown;          // [G][2][B][UMAX]
  float* gpown;         // [G][B][C2]
  float4* partv;        // [B][G]
  float4* partd;        // [B][G] (unused: duration argmax goes through dmax)
  unsigned long long* amax;  // [2][B] packed (orderable logit, ~index) token argmax per step parity
  unsigned long long* dmax;  // [2][B] same for the duration head
  unsigned long long* prof;  // optional [16] phase times (ns) of CTA 0
  int* tokens;
  int* frames;
  float* scores;
  int* durs;
  int* counts;
  Ctrl* ctrl;
  unsigned* bar;        // grid barrier word
};

__host__ __device__ inline int own_lo(int n, int c, int G) { return (int)((long long)n * c / G); }

// Shared memory: [weights][per-warp activation slots, reused as the
// reduction scratch][per-row control][mbarriers]
struct Smem {
  float* w;
  float* ring;   // NCW slots of slotk x 32 floats
  float* red;    // overlays ring
  int* label;
  int* tb;
  int* ub;
  int* flag;     // bit0 done(FS) / inactive(LL), bit1 accepted this step
  int* kdec;
  float* vdec;
  int* ddec;
  int* cnt;      // emitted count per row (replicated; the owner writes global counts)
  int* misc;     // [2]=t, [3]=sym, [4]=par
  float* own;    // own-state (hh0 [B][C1], c [2][B][umax], gp [B][C2]) when own_smem
  unsigned long long* prof;  // [16] phase-time accumulators (CTA 0, thread 0)
  uint64_t* full;  // one per warp
  uint64_t* wbar;
};

__host__ __device__ inline size_t ring_floats(int ns) {
  const size_t r = (size_t)NCW * ns * 8 * RB;
  return r > (size_t)RED_FLOATS ? r : (size_t)RED_FLOATS;
}

__host__ __device__ inline size_t own_floats(int B, int umax) {
  return (size_t)B * C1 + 2 * (size_t)B * umax + (size_t)B * C2;
}

__host__ __device__ inline size_t smem_bytes(int wfloats, int ns, int B, size_t ownf = 0) {
  size_t b = (size_t)wfloats * 4 + ring_floats(ns) * 4;
  b += (size_t)B * 4 * 8 + 64 + ownf * 4 + 16 * 8;
  b = (b + 15) / 16 * 16;
  b += 8 * (NCW + 1);
  return b;
}

__device__ inline Smem carve_p(unsigned char* base, const PParams& P) {
  Smem s;
  s.w = reinterpret_cast<float*>(base);
  s.ring = s.w + P.wfloats;
  s.red = s.ring;
  int* ip = reinterpret_cast<int*>(s.ring + ring_floats(P.ns));
  s.label = ip;
  s.tb = ip + P.B;
  s.ub = ip + 2 * P.B;
  s.flag = ip + 3 * P.B;
  s.kdec = ip + 4 * P.B;
  s.vdec = reinterpret_cast<float*>(ip + 5 * P.B);
  s.ddec = ip + 6 * P.B;
  s.cnt = ip + 7 * P.B;
  s.misc = ip + 8 * P.B;
  s.own = reinterpret_cast<float*>(s.misc + 16);
  const size_t ownf = P.own_smem ? own_floats(P.B, P.cell == 1 ? UMAX_LSTM : UMAX_TANH) : 0;
  size_t off = (size_t)(reinterpret_cast<unsigned char*>(s.own + ownf) - base);
  off = (off + 15) / 16 * 16;
  s.prof = reinterpret_cast<unsigned long long*>(base + off);
  off += 16 * 8;
  s.full = reinterpret_cast<uint64_t*>(base + off);
  s.wbar = s.full + NCW;
  return s;
}

// ------------------------------------------------------------ grid barrier
// Split arrive / wait on one word: the master CTA adds 0x80000000-(G-1),
// the others 1, so bit 31 flips when the last CTA arrives (the algorithm of
// cooperative_groups' grid sync: 1.2 us on B200 vs 2.5 us for a
// count+generation pair, scripts/microbench.cu), with independent work
// allowed between the two halves.
__device__ __forceinline__ unsigned bar_arrive(unsigned* bar, int G) {
  // order generic-proxy global stores before other CTAs' bulk-copy reads
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __syncthreads();
  unsigned old = 0;
  if (threadIdx.x == 0) {
    const unsigned nb = blockIdx.x == 0 ? 0x80000000u - (unsigned)(G - 1) : 1u;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(nb) : "memory");
  }
  return old;
}

__device__ __forceinline__ void bar_wait(unsigned* bar, unsigned old) {
  if (threadIdx.x == 0) {
    unsigned cur;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
    } while (((old ^ cur) & 0x80000000u) == 0);
  }
  __syncthreads();
}

__device__ __forceinline__ void grid_barrier(unsigned* bar, int G) { bar_wait(bar, bar_arrive(bar, G)); }

// ------------------------------------------------------------ activations
// Element (row b, feature k) of a k-major activation buffer with K features:
// [rb][K][32 rows], the row index XOR-swizzled by (k & 3) << 3 so a warp's
// LDS.128 of 8 row quads x 4 consecutive k hit 8 distinct bank quads per k.
// Any contiguous feature range is one contiguous block -> one bulk copy.
__device__ __forceinline__ size_t act_idx(int b, int k, int K) {
  const int rb = b >> 5, r = b & 31;
  return ((size_t)rb * K + k) * RB + (r ^ ((k & 3) << 3));
}

// 64-bit key whose unsigned max is the lowest-index argmax of float values:
// (order-preserving float bits << 32) | (~index).  Merged with red.max.u64,
// which is order-independent, so the decision stays deterministic.
__device__ __forceinline__ unsigned long long argmax_key(float v, int idx) {
  unsigned u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)u << 32) | (unsigned long long)(0xffffffffu - (unsigned)idx);
}
__device__ __forceinline__ int argmax_key_index(unsigned long long k) {
  return (int)(0xffffffffu - (unsigned)(k & 0xffffffffull));
}

__device__ __forceinline__ void store_act(float* buf, int b, int k, int K, float v) {
  buf[act_idx(b, k, K)] = v;
}

// A source for a GEMV pass: up to two concatenated buffers (features K0 + K1).
struct ASrc {
  const float* a0;
  int k0;
  const float* a1;
  int k1;
};

// acc[i][c] += A[k][4rq+i] * W[k][c] for one k of this lane.
template <int C>
__device__ __forceinline__ void mac_step(const float4 a, const float* wr, float (&acc)[4][C]) {
#pragma unroll
  for (int q = 0; q < C / 4; ++q) {
    const float4 w = lds4(wr + 4 * q);
    acc[0][4 * q + 0] = fmaf(a.x, w.x, acc[0][4 * q + 0]);
    acc[0][4 * q + 1] = fmaf(a.x, w.y, acc[0][4 * q + 1]);
    acc[0][4 * q + 2] = fmaf(a.x, w.z, acc[0][4 * q + 2]);
    acc[0][4 * q + 3] = fmaf(a.x, w.w, acc[0][4 * q + 3]);
    acc[1][4 * q + 0] = fmaf(a.y, w.x, acc[1][4 * q + 0]);
    acc[1][4 * q + 1] = fmaf(a.y, w.y, acc[1][4 * q + 1]);
    acc[1][4 * q + 2] = fmaf(a.y, w.z, acc[1][4 * q + 2]);
    acc[1][4 * q + 3] = fmaf(a.y, w.w, acc[1][4 * q + 3]);
    acc[2][4 * q + 0] = fmaf(a.z, w.x, acc[2][4 * q + 0]);
    acc[2][4 * q + 1] = fmaf(a.z, w.y, acc[2][4 * q + 1]);
    acc[2][4 * q + 2] = fmaf(a.z, w.z, acc[2][4 * q + 2]);
    acc[2][4 * q + 3] = fmaf(a.z, w.w, acc[2][4 * q + 3]);
    acc[3][4 * q + 0] = fmaf(a.w, w.x, acc[3][4 * q + 0]);
    acc[3][4 * q + 1] = fmaf(a.w, w.y, acc[3][4 * q + 1]);
    acc[3][4 * q + 2] = fmaf(a.w, w.z, acc[3][4 * q + 2]);
    acc[3][4 * q + 3] = fmaf(a.w, w.w, acc[3][4 * q + 3]);
  }
}

// Reduce acc over the 4 ks lanes and the 8 warps.  Across ks a butterfly
// reduce-scatter (2C + C shuffles instead of 8C for an all-reduce) leaves lane
// ks holding row 4rq+ks's C sums; every warp then writes them to
// sm.red[warp][32][C] and red_sum adds the 8 warps in fixed order.
// red overlays the activation slots, so everyone must be done with them.
template <int C>
__device__ __forceinline__ void reduce_tile(const Smem& sm, float (&acc)[4][C]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rq = lane >> 2, ks = lane & 3;
  const bool hi2 = (ks & 2) != 0, hi1 = (ks & 1) != 0;
  float h[2][C];  // step A (partner lane ^ 2): keep rows {0,1} or {2,3}
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const float keep = hi2 ? acc[2 + i][c] : acc[i][c];
      const float send = hi2 ? acc[i][c] : acc[2 + i][c];
      h[i][c] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
  float q[C];  // step B (partner lane ^ 1): keep row (ks & 1) of the pair
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const float keep = hi1 ? h[1][c] : h[0][c];
    const float send = hi1 ? h[0][c] : h[1][c];
    q[c] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
  }
  __syncthreads();  // all warps are done reading their activation slots
  float* dst = sm.red + ((size_t)warp * RB + 4 * rq + ks) * C;
#pragma unroll
  for (int c = 0; c < C; c += 4) *reinterpret_cast<float4*>(dst + c) = make_float4(q[c], q[c + 1], q[c + 2], q[c + 3]);
  __syncthreads();
}

__device__ __forceinline__ float red_sum(const Smem& sm, int r, int c, int C) {
  const float* red = sm.red + r * C + c;
  const int ws = RB * C;
  return ((red[0] + red[ws]) + (red[2 * ws] + red[3 * ws])) +
         ((red[4 * ws] + red[5 * ws]) + (red[6 * ws] + red[7 * ws]));
}

// One GEMV pass over an activation source for every row block:
// out[32 rows][C] = A[32][K] @ W[K][C], W resident in smem ([K][C]).
// Warp w owns the contiguous feature slice [w*K/8, (w+1)*K/8) and streams it
// through its own slot with one bulk copy per ns*8 features (bulk copies
// from one warp serialise, so every warp issues its own:
// scripts/microbench3.cu).  Lane (rq, ks): rows 4rq..4rq+3, features
// k = 4j + ks of each slot.  epi(rb) runs after the block reduction.
template <int C, typename Epi>
__device__ __forceinline__ void gemv_pass(const Smem& sm, const PParams& P, unsigned& ph,
                                          const ASrc& A, const float* W, Epi epi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rq = lane >> 2, ks = lane & 3;
  const int K = A.k0 + A.k1, kw = K / NCW, kbeg = warp * kw;
  const int slotk = P.ns * 8;
  float* slot = sm.ring + (size_t)warp * slotk * RB;
  uint64_t* bar = &sm.full[warp];
  const bool seg0 = kbeg < A.k0;
  const float* base = seg0 ? A.a0 : A.a1;
  const int kseg = seg0 ? A.k0 : A.k1;
  const int koff = seg0 ? kbeg : kbeg - A.k0;
  const int aoff = (4 * rq) ^ (ks << 3);
  for (int rb = 0; rb < P.nrb; ++rb) {
    float acc[4][C];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < C; ++c) acc[i][c] = 0.0f;
    for (int kk = 0; kk < kw; kk += slotk) {
      const int nk = kw - kk < slotk ? kw - kk : slotk;
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(bar, (uint32_t)(nk * RB * 4));
        bulk_g2s(slot, base + ((size_t)rb * kseg + koff + kk) * RB, (uint32_t)(nk * RB * 4), bar);
      }
      unsigned long long tq0 = 0;
      if (P.prof && blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tq0));
      mbar_wait(bar, ph);
      ph ^= 1u;
      if (P.prof && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long tq1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tq1));
        sm.prof[13] += tq1 - tq0;
        sm.prof[14] += 1;
      }
      const float* wk = W + (size_t)(kbeg + kk + ks) * C;
#pragma unroll 4
      for (int j = 0; j < nk / 4; ++j) {
        const float4 a = lds4(slot + (4 * j + ks) * RB + aoff);
        mac_step<C>(a, wk + (size_t)4 * j * C, acc);
      }
      __syncwarp();
    }
    unsigned long long tr0 = 0;
    if (P.prof && blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr0));
    reduce_tile<C>(sm, acc);
    epi(rb);
    __syncthreads();
    if (P.prof && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long tr1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr1));
      sm.prof[15] += tr1 - tr0;
    }
  }
}

// ------------------------------------------------------------ the kernel
__global__ void __launch_bounds__(NTH, 1) persistent_kernel(PParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem sm = carve_p(smem_raw, P);
  const int cta = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = P.G, B = P.B;
  const bool lstm = P.cell == 1;
  const int umax = lstm ? UMAX_LSTM : UMAX_TANH;
  const int u0 = own_lo(P.H, cta, G), u1 = own_lo(P.H, cta + 1, G);
  const int nu = u1 - u0;                          // owned units
  const int p0 = own_lo(P.J, cta, G), p1 = own_lo(P.J, cta + 1, G);
  const int n0 = own_lo(P.NJ, cta, G), n1 = own_lo(P.NJ, cta + 1, G);
  const int blank = P.V1 - 1;
  const bool fs = P.algo == ALGO_FS, tdt = P.algo == ALGO_TDT;
  float* hh0own = P.own_smem ? sm.own : P.hh0own + (size_t)cta * B * C1;
  float* cown = P.own_smem ? sm.own + (size_t)B * C1 : P.cown + (size_t)cta * 2 * B * umax;
  float* gpown = P.own_smem ? sm.own + (size_t)B * C1 + 2 * (size_t)B * umax
                            : P.gpown + (size_t)cta * B * C2;
  const float* bias = P.bias + (size_t)cta * 2 * C1;

  // ---- one-time setup: barriers, resident weights, control state ----
  if (tid == 0) {
    for (int i = 0; i < NCW; ++i) mbar_init(&sm.full[i], 1);
    mbar_init(sm.wbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    const size_t bytes = (size_t)P.wfloats * 4;
    mbar_arrive_expect_tx(sm.wbar, (uint32_t)bytes);
    const float* src = P.wpack + (size_t)cta * P.wfloats;
    for (size_t o = 0; o < bytes; o += 32768) {
      const uint32_t nb = (uint32_t)(bytes - o < 32768 ? bytes - o : 32768);
      bulk_g2s(reinterpret_cast<unsigned char*>(sm.w) + o,
               reinterpret_cast<const unsigned char*>(src) + o, nb, sm.wbar);
    }
  }
  int maxlen = 0;
  for (int b = tid; b < B; b += NTH) {
    sm.label[b] = blank;
    sm.tb[b] = 0;
    sm.ub[b] = 0;
    const int len = P.out_len[b];
    sm.flag[b] = (fs ? (0 >= len) : !(0 < len)) | 2;  // accept all for P0
    sm.cnt[b] = 0;
    if (b % G == cta) P.counts[b] = 0;
    if (cta == 0) {
      P.amax[b] = 0ull;
      P.amax[B + b] = 0ull;
      P.dmax[b] = 0ull;
      P.dmax[B + b] = 0ull;
    }
  }
  for (int b = 0; b < B; ++b) maxlen = max(maxlen, __ldg(&P.out_len[b]));
  // zero own state: h0/h1 (both parities) for owned units, c, hh0 (= 0 @ W), gp
  for (int i = tid; i < B * nu; i += NTH) {
    const int b = i / nu, u = u0 + i % nu;
    store_act(P.h0, b, u, P.Hp, 0.0f);
    store_act(P.h1[0], b, u, P.Hp, 0.0f);
    store_act(P.h1[1], b, u, P.Hp, 0.0f);
  }
  for (int i = tid; i < 2 * B * umax; i += NTH) cown[i] = 0.0f;
  for (int i = tid; i < B * C1; i += NTH) hh0own[i] = 0.0f;
  for (int i = tid; i < B * C2; i += NTH) gpown[i] = 0.0f;
  if (tid == 0) {
    sm.misc[2] = 0;  // t
    sm.misc[3] = 0;  // sym
    sm.misc[4] = 0;  // par
  }
  mbar_wait(sm.wbar, 0);
  const float* Whh0 = sm.w + P.off_hh0;
  const float* W1 = sm.w + P.off_w1;
  const float* Wpp = sm.w + P.off_pp;
  const float* WJ = sm.w + P.off_j;
  unsigned ph = 0;  // this warp's slot mbarrier phase
  long long joint_evals = 0, pred_steps = 0, outer_iters = 0, iters = 0;
  unsigned long long t_last = 0;
  if (tid < 16) sm.prof[tid] = 0ull;
  auto mark = [&](int id) {
    if (P.prof && cta == 0 && tid == 0) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (t_last) sm.prof[id] += now - t_last;
      t_last = now;
    }
  };
  int err = 0;
  __syncthreads();

  // ---- layer-0 cell for owned units (accepted rows) ----
  // gates = (table0[label] + hh0) + b   (model.cpp:48 order; App. B)
  auto cell0 = [&]() {
    const int G4 = P.Gg;
    for (int i = tid; i < B * nu; i += NTH) {
      const int b = i / nu, lu = i % nu, u = u0 + lu;
      if (!(sm.flag[b] & 2)) continue;
      const int lab = sm.label[b];
      if (lstm) {
        float g4[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const float ih = __ldg(&P.table0[(size_t)lab * P.GH + u * G4 + g]);
          g4[g] = (ih + hh0own[b * C1 + lu * 4 + g]) + bias[lu * 4 + g];
        }
        const float c_old = cown[b * umax + lu];
        const float i_ = sigmoid_f(g4[0]), f_ = sigmoid_f(g4[1]);
        const float g_ = tanhf(g4[2]), o_ = sigmoid_f(g4[3]);
        const float cn = f_ * c_old + i_ * g_;
        cown[b * umax + lu] = cn;
        store_act(P.h0, b, u, P.Hp, o_ * tanhf(cn));
      } else {
        const float ih = __ldg(&P.table0[(size_t)lab * P.GH + u]);
        store_act(P.h0, b, u, P.Hp, tanhf((ih + hh0own[b * C1 + lu]) + bias[lu]));
      }
    }
  };

  // ---- trunk = relu(fp[b, t_b] + gp) for owned joint-input columns ----
  auto refresh_trunk = [&](bool gp_fresh) {
    (void)gp_fresh;
    const int np = p1 - p0;
    for (int i = tid; i < B * np; i += NTH) {
      const int b = i / np, lj = i % np, j = p0 + lj;
      int t = fs ? sm.misc[2] : sm.tb[b];
      t = t < 0 ? 0 : (t > P.T - 1 ? P.T - 1 : t);
      const float f = __ldg(&P.fp[((size_t)b * P.T + t) * P.Jp + j]);
      store_act(P.trunk, b, j, P.Jp, fmaxf(f + gpown[b * C2 + lj], 0.0f));
    }
  };

  // ---- the prediction step for accepted rows (after decisions) ----
  auto pred_step = [&]() {
    mark(2);
    cell0();
    mark(3);
    grid_barrier(P.bar, G);
    mark(4);
    const int par = sm.misc[4];
    if (P.L == 2) {
      // layer 1: [h0' | h1] @ W_1, fused LSTM cell; h1 ping-pong
      {
        ASrc A{P.h0, P.Hp, P.h1[par], P.Hp};
        gemv_pass<C1>(sm, P, ph, A, W1, [&](int rb) {
          for (int o = tid; o < RB * nu; o += 256) {
            const int r = o / nu, lu = o % nu, b = rb * RB + r, u = u0 + lu;
            if (b >= B) continue;
            float hn;
            if (sm.flag[b] & 2) {
              float g4[4];
#pragma unroll
              for (int g = 0; g < 4; ++g) g4[g] = red_sum(sm, r, lu * 4 + g, C1) + bias[C1 + lu * 4 + g];
              const float c_old = cown[(B + b) * umax + lu];
              const float i_ = sigmoid_f(g4[0]), f_ = sigmoid_f(g4[1]);
              const float g_ = tanhf(g4[2]), o_ = sigmoid_f(g4[3]);
              const float cn = f_ * c_old + i_ * g_;
              cown[(B + b) * umax + lu] = cn;
              hn = o_ * tanhf(cn);
            } else {
              hn = P.h1[par][act_idx(b, u, P.Hp)];
            }
            store_act(P.h1[par ^ 1], b, u, P.Hp, hn);
          }
        });
      }
      __syncthreads();
      mark(6);
      if (tid == 0) sm.misc[4] = par ^ 1;
      // arrive; the next step's h0' @ W_hh0 needs no other CTA -> hides the barrier
      const unsigned ticket = bar_arrive(P.bar, G);
      // hh0 for the next step: h0' @ W_hh0 (owned gate columns)
      {
        ASrc A{P.h0, P.Hp, nullptr, 0};
        gemv_pass<C1>(sm, P, ph, A, Whh0, [&](int rb) {
          for (int o = tid; o < RB * C1; o += 256) {
            const int r = o / C1, c = o % C1, b = rb * RB + r;
            if (b < B && (sm.flag[b] & 2)) hh0own[b * C1 + c] = red_sum(sm, r, c, C1);
          }
        });
      }
      mark(5);
      bar_wait(P.bar, ticket);
      mark(7);
      // pred_proj over h1', trunk
      {
        ASrc A{P.h1[par ^ 1], P.Hp, nullptr, 0};
        gemv_pass<C2>(sm, P, ph, A, Wpp, [&](int rb) {
          const int np = p1 - p0;
          for (int o = tid; o < RB * np; o += 256) {
            const int r = o / np, lj = o % np, b = rb * RB + r;
            if (b < B && (sm.flag[b] & 2)) gpown[b * C2 + lj] = red_sum(sm, r, lj, C2);
          }
        });
      }
    } else {
      // one layer: pred_proj over h0' plus the next step's hh0 (same chunks)
      ASrc A{P.h0, P.Hp, nullptr, 0};
      gemv_pass<C1>(sm, P, ph, A, Whh0, [&](int rb) {
        for (int o = tid; o < RB * C1; o += 256) {
          const int r = o / C1, c = o % C1, b = rb * RB + r;
          if (b < B && (sm.flag[b] & 2)) hh0own[b * C1 + c] = red_sum(sm, r, c, C1);
        }
      });
      gemv_pass<C2>(sm, P, ph, A, Wpp, [&](int rb) {
        const int np = p1 - p0;
        for (int o = tid; o < RB * np; o += 256) {
          const int r = o / np, lj = o % np, b = rb * RB + r;
          if (b < B && (sm.flag[b] & 2)) gpown[b * C2 + lj] = red_sum(sm, r, lj, C2);
        }
      });
    }
    __syncthreads();
    mark(8);
    refresh_trunk(true);
    ++pred_steps;
    mark(9);
    grid_barrier(P.bar, G);
    mark(10);
  };

  // prologue: P0 = pred(blank, 0) for every row (decoders.cpp:414-430)
  pred_step();
  for (int b = tid; b < B; b += NTH) sm.flag[b] &= ~2;
  __syncthreads();
  bool running = fs ? (maxlen > 0) : false;
  if (!fs) {
    int any = 0;
    for (int b = 0; b < B; ++b) any |= !(sm.flag[b] & 1);
    running = any;
  }

  while (running) {
    const int jpar = (int)(joint_evals & 1);
    // ---- J: joint logits for owned columns -> per-CTA partials ----
    {
      ASrc A{P.trunk, P.Jp, nullptr, 0};
      gemv_pass<C2>(sm, P, ph, A, WJ, [&](int rb) {
        // half-warp per row: lanes 0..7 hold the 8 columns
        const int nn = n1 - n0;
        for (int r = (tid >> 3); r < RB; r += 32) {
          const int b = rb * RB + r, l8 = tid & 7;
          const int n = n0 + l8;
          const float x = l8 < nn ? red_sum(sm, r, l8, C2) : -INFINITY;
          const bool isv = l8 < nn && n < P.V1, isd = l8 < nn && n >= P.V1;
          float mv = isv ? x : -INFINITY, md = isd ? x : -INFINITY;
#pragma unroll
          for (int o = 4; o >= 1; o >>= 1) {
            mv = fmaxf(mv, __shfl_xor_sync(0xffffffffu, mv, o));
            md = fmaxf(md, __shfl_xor_sync(0xffffffffu, md, o));
          }
          float ev = isv ? expf(x - mv) : 0.0f, ed = isd ? expf(x - md) : 0.0f;
          float bv = isv ? x : -INFINITY, bd = isd ? x : -INFINITY;
          int iv = isv ? n : 0x7fffffff, id = isd ? n - P.V1 : 0x7fffffff;
#pragma unroll
          for (int o = 4; o >= 1; o >>= 1) {
            ev += __shfl_xor_sync(0xffffffffu, ev, o);
            ed += __shfl_xor_sync(0xffffffffu, ed, o);
            const float obv = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oiv = __shfl_xor_sync(0xffffffffu, iv, o);
            if (obv > bv || (obv == bv && oiv < iv)) {
              bv = obv;
              iv = oiv;
            }
            const float obd = __shfl_xor_sync(0xffffffffu, bd, o);
            const int oid = __shfl_xor_sync(0xffffffffu, id, o);
            if (obd > bd || (obd == bd && oid < id)) {
              bd = obd;
              id = oid;
            }
          }
          if (l8 == 0 && b < B) {
            P.partv[(size_t)b * G + cta] = make_float4(mv, ev, bv, __int_as_float(iv));
            if (bv != -INFINITY) atomicMax(&P.amax[jpar * B + b], argmax_key(bv, iv));
            if (P.D && bd != -INFINITY) atomicMax(&P.dmax[jpar * B + b], argmax_key(bd, id));
          }
        }
      });
    }
    ++joint_evals;
    ++iters;
    mark(0);
    grid_barrier(P.bar, G);
    mark(1);

    // ---- D: decisions (identical in every CTA) ----
    // The argmax of every row (argmax_last_into, tensor.cpp:268-312: lowest
    // index on ties) arrives merged in amax/dmax; every CTA reads them and
    // applies the same rules.  Only the owner CTA of a row (b mod G) merges
    // that row's per-CTA (max, sumexp) partials into lse (log_softmax_into,
    // tensor.cpp:463-480) for the emitted score and writes the emission.
    {
      // argmax reads by the high warps, lse merges by the low warps: the two
      // L2 round trips overlap
      for (int b = NTH - 1 - tid; b >= 0 && b < B; b -= NTH) {
        sm.kdec[b] = argmax_key_index(__ldcg(&P.amax[jpar * B + b]));
        sm.ddec[b] = P.D ? P.durations[argmax_key_index(__ldcg(&P.dmax[jpar * B + b]))] : 0;
      }
      if (cta == 0)
        for (int b = tid; b < B; b += NTH) {
          P.amax[(jpar ^ 1) * B + b] = 0ull;
          if (P.D) P.dmax[(jpar ^ 1) * B + b] = 0ull;
        }
      {
        const int warp = tid >> 5, lane = tid & 31;
        for (int b = cta + G * warp; b < B; b += G * NCW) {
          float Mx = -INFINITY, Sx = 0.0f, best = -INFINITY;
          for (int c = lane; c < G; c += 32) {
            const float4 p = __ldcg(&P.partv[(size_t)b * G + c]);
            if (p.x != -INFINITY) {
              const float nm = fmaxf(Mx, p.x);
              Sx = (Sx == 0.0f ? 0.0f : Sx * expf(Mx - nm)) + p.y * expf(p.x - nm);
              Mx = nm;
              best = fmaxf(best, p.z);
            }
          }
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) {
            const float om = __shfl_xor_sync(0xffffffffu, Mx, o);
            const float os = __shfl_xor_sync(0xffffffffu, Sx, o);
            best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
            const float nm = fmaxf(Mx, om);
            Sx = (Sx == 0.0f ? 0.0f : Sx * expf(Mx - nm)) + (os == 0.0f ? 0.0f : os * expf(om - nm));
            Mx = nm;
          }
          if (lane == 0) sm.vdec[b] = best - (Mx + logf(Sx));
        }
      }
      __syncthreads();
      // decision rules (thread per row), decoders.cpp:261-307 / 432-512
      int acc_any = 0, live_any = 0;
      const int t_fs = sm.misc[2];
      for (int b = tid; b < B; b += NTH) {
        int f = sm.flag[b] & ~2;
        const int k = sm.kdec[b];
        const float v = sm.vdec[b];
        if (fs) {
          if (!(f & 1)) {
            if (k == blank) {
              f |= 1;
            } else {
              if (b % G == cta) {
                const int nb = sm.cnt[b];
                if (nb < P.cap) {
                  const size_t o = (size_t)b * P.cap + nb;
                  P.tokens[o] = k;
                  P.frames[o] = t_fs;
                  P.scores[o] = v;
                  P.durs[o] = 0;
                  P.counts[b] = nb + 1;
                }
              }
              sm.cnt[b] += 1;
              sm.label[b] = k;
              f |= 2;
            }
          }
          live_any |= !(f & 1);
        } else if (!(f & 1)) {
          const int len = __ldg(&P.out_len[b]);
          int t = sm.tb[b], u = sm.ub[b];
          if (k == blank) {
            const int d = tdt ? sm.ddec[b] : 1;
            t += d > 1 ? d : 1;
            u = 0;
          } else {
            const int d = tdt ? sm.ddec[b] : 0;
            if (b % G == cta) {
              const int nb = sm.cnt[b];
              if (nb < P.cap) {
                const size_t o = (size_t)b * P.cap + nb;
                P.tokens[o] = k;
                P.frames[o] = t;
                P.scores[o] = v;
                P.durs[o] = d;
                P.counts[b] = nb + 1;
              }
            }
            sm.cnt[b] += 1;
            sm.label[b] = k;
            f |= 2;
            u += 1;
            if (d > 0) {
              t += d;
              u = 0;
            } else if (u == P.ms) {
              t += 1;
              u = 0;
            }
          }
          sm.tb[b] = t;
          sm.ub[b] = u;
          if (!(t < len)) f |= 1;
          live_any |= !(f & 1);
        }
        acc_any |= (f >> 1) & 1;
        sm.flag[b] = f;
      }
      acc_any = __syncthreads_or(acc_any);
      live_any = __syncthreads_or(live_any);
      bool finish = false;
      if (fs) {
        int sym = sm.misc[3] + 1;
        int t = t_fs;
        if (!live_any || sym >= P.ms) {  // frame ends (decoders.cpp:297-313)
          t += 1;
          sym = 0;
          ++outer_iters;
          if (t >= maxlen) finish = true;
          __syncthreads();
          for (int b = tid; b < B; b += NTH)
            sm.flag[b] = (sm.flag[b] & 2) | (t >= __ldg(&P.out_len[b]) ? 1 : 0);
        }
        __syncthreads();
        if (tid == 0) {
          sm.misc[3] = sym;
          sm.misc[2] = t;
        }
        __syncthreads();
      } else {
        finish = !live_any;
      }
      if (iters > P.max_iters) {
        err = ERR_RUNAWAY;
        finish = true;
      }
      if (finish) break;
      if (acc_any) {
        pred_step();
        if (!fs) ++outer_iters;
      } else {
        refresh_trunk(false);
        mark(11);
        grid_barrier(P.bar, G);
        mark(12);
      }
      for (int b = tid; b < B; b += NTH) sm.flag[b] &= ~2;
      __syncthreads();
    }
  }
  if (P.prof && cta == 0 && tid < 16) P.prof[tid] += sm.prof[tid];
  if (cta == 0 && tid == 0) {
    Ctrl* c = P.ctrl;
    c->joint_evals = joint_evals;
    c->pred_steps = pred_steps;
    c->outer_iters = outer_iters;
    c->iters = iters;
    c->err = err;
  }
}

}  // namespace pk
}  // namespace rnntg
