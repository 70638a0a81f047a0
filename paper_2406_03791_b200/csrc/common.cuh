// common.cuh — device-side layouts, control block and PTX helpers shared by
// the decoder kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rnntg {

constexpr int RB = 32;      // batch rows per row block (one tile of the step GEMVs)
constexpr int CT = 16;      // output columns per step-GEMV tile
constexpr int NW = 8;       // warps per step CTA (split K)
constexpr int NT = NW * 32; // threads per step CTA
constexpr int MAXL = 4;     // max prediction-network layers
constexpr int MAXD = 16;    // max duration classes
constexpr int MAXRB = 32;   // max row blocks (batch <= 1024)

enum Algo { ALGO_FS = 0, ALGO_LL = 1, ALGO_TDT = 2 };
enum Err { ERR_NONE = 0, ERR_RUNAWAY = 7 };

// Device weights after repacking.  Padded extents are multiples of 32 so
// every row starts 128-byte aligned and every k-slice splits evenly over
// the NW warps.  Gate columns are interleaved per unit (col = u*G + gate) so
// one CTA tile holds all gates of its units and fuses the cell update.
struct DevModel {
  int V1, E, H, Hp, L, cell, G, GH;  // GH = G*Hp gate columns
  int J, Jp, F, Fp, D;
  int V1p;   // vocab columns padded to CT
  int NOUT;  // V1p + (D ? CT : 0): out_proj || dur_proj columns
  int NCH;   // vocab chunks (V1p / CT)
  int NCHT;  // + duration chunk
  int durations[MAXD];
  const float* table0;          // [V1][GH]   embedding @ W_ih0 (exact, sequential k)
  const float* w[MAXL];         // tiled [GH/16][K][16]; K = Hp (W_hh0) or 2Hp ([W_ih;W_hh])
  const float* bias[MAXL];      // [GH]
  const float* pred_proj;       // tiled [Jp/16][Hp][16]
  const float* out_ext;         // tiled [NOUT/16][Jp][16] (out_proj || dur_proj)
  const float* enc;             // [Fp][Jp]
  const float* enc_hi;          // tcgen05 operands: enc^T split into tf32 hi/lo,
  const float* enc_lo;          // K-major [Jp][Fp]
  // RNNTG_CELL_SCRIPTED tables (rnntg_model_create_scripted)
  const int* s_lab;   // [s_B][s_T][s_U]
  const int* s_fsarr; // [s_B][s_T + 1]
  const int* s_darr;  // [s_B][s_T]
  const int* s_dval;  // [s_B][s_T][s_U + 1]
  int s_B, s_T, s_U;
};

// Loop/scalar control block (device memory, one per decoder).
struct Ctrl {
  int t;        // frame index (frame-sync)
  int sym;      // symbols emitted at this frame (frame-sync)
  int max_len;  // max(out_len)
  int par;      // ping-pong parity of the prediction state buffers
  int err;
  int abort;
  int any;
  int pad0;
  unsigned ctr_joint_rb[MAXRB];
  unsigned ctr_joint_all;
  unsigned ctr_pp;
  unsigned pad1[2];
  long long joint_evals;
  long long pred_steps;
  long long outer_iters;
  long long iters;
};

struct DevState {
  int B, Bp, nrb, T, ms, cap, algo, use_cond;
  long long max_iters;
  const float* x;        // [B,T,F] (user layout)
  const int* out_len;    // [B]
  float* fp;             // [B*T][Jp] encoder projection (K1 output)
  float* h[MAXL][2];     // [Bp][Hp] per layer, ping-pong
  float* c[MAXL][2];
  float* gp;             // [Bp][Jp] cached predictor projection
  int* last_label;
  int* accept;           // row accepted a label this step -> run / commit pred
  int* done;             // frame-sync blank mask
  int* need;             // label-loop: row still needs a decision this round
  int* active;           // label-loop: t_row < out_len
  int* t_row;
  int* u_row;
  int* counts;
  int* tokens;           // [B][cap]
  int* frames;
  float* scores;
  int* durs;
  float4* part;          // [Bp][NCHT] per-chunk (max, sumexp, best, idx)
  Ctrl* ctrl;
  cudaGraphConditionalHandle h_outer, h_inner;
  float* dbg_logits;     // [Bp][NOUT] (step API only)
  float* dbg_lse;        // [2*Bp]
};

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// 1-D bulk copy global -> shared (TMA engine), completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Programmatic dependent launch controls.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ float4 ldg4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ float4 lds4(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}

// Coherent (L2) load for flags and counters written by other CTAs.
__device__ __forceinline__ int ld_volatile(const int* p) { return __ldcg(p); }

__device__ __forceinline__ float sigmoid_f(float x) { return 1.0f / (1.0f + expf(-x)); }

}  // namespace rnntg
