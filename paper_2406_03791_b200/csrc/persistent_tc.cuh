// persistent_tc.cuh — K6: the tensor-core persistent decoder.
//
// The whole greedy decode (frame-looping, label-looping, TDT label-looping)
// runs in ONE cooperative kernel whose CTAs are specialised by ROLE, one
// 128-row weight tile each, and pass activations to each other through
// per-chunk dataflow counters in global memory (no grid barriers):
//
//   role   weights (swap-AB: M = 128 output rows)   input        output
//   J      [out_proj || dur_proj] cols 128t..        trunk(s)     per-row argmax words, (max, sumexp)
//   P      pred_proj cols 128t..                     h_{L-1}(p)   gp -> trunk(s+1) = relu(fp + gp)
//   R_0    W_hh0 gate rows (unit-major, 32 units)    table0[k] + hh0(p) (registers): the layer-0 cell
//                                                    -> h_0(p+1); then h_0(p+1) @ W_hh0 -> hh0(p+2)
//   R_l    W_hh_l gate rows, l >= 1                  h_l(p)       hh_l(p+1) -> global (for I_l);
//                                                                 R_{L-1} tile 0 also merges the J
//                                                                 partials: scores, hypotheses
//   I_l    W_ih_l gate rows, l >= 1                  h_{l-1}(p)   (+ hh_l) cell -> h_l(p)
//
// Row groups.  The batch is split into ngrp <= 8 groups of <= 32 rows; every
// CTA serves every group, visiting the live groups round-robin one step
// ("item") at a time.  The groups are independent decodes (model.hpp:89-91)
// with their own buffers, counters and replicated control, so while one
// group's step is in flight down the chain (J -> decision -> R_0 -> I_1 -> P),
// the CTAs that are done with it work on the next group's step.
//
// Arithmetic.  Every GEMV is D[128 x 32 rows] = W[128 x K] . A^T on the
// 5th-gen tensor cores (tcgen05.mma.kind::f16, fp32 accumulate) with an
// fp16 hi/lo split of BOTH operands: W' = W*2^s = W_hi + W_lo, A = A_hi + A_lo,
// D = W_hi.[A_hi | A_lo] (one MMA, N = 64) + W_lo.A_hi (N = 32), i.e. all
// products down to 2^-22 relative (~fp32; the dropped W_lo.A_lo is 2^-22).
// W_hi is resident in TENSOR memory (the MMA's A operand read from TMEM),
// W_lo in shared memory (SWIZZLE_128B K-major) except its first
// nlo_chunks(KC) chunks, which fit in TMEM too; a 128 x 640 tile (320 KB of
// fp16 pairs) stays on chip for the whole decode.
//
// Activations move as fp16 hi/lo images already in the UMMA canonical
// layout ([64 rows = 32 hi + 32 lo][64 k] chunks of 8 KB, 128B-swizzled by
// the TMA tensor map), so a consumer's load is one tensor copy per chunk.  A
// chunk is published by its producers (TMA store, wait_group, proxy fence,
// release) with an add on its counter; consumers poll the counter (relaxed,
// then one acquire re-read) and stream chunks into a 4-stage ring as they
// appear, overlapping the transfer with the MMAs of earlier chunks.
//
// Control state (labels, cursors, masks, frame counters) is replicated in
// every CTA: each CTA merges the J tiles' argmax words for every row and
// applies the same decision rules (decoders.cpp:261-307, 432-512), so no
// decision broadcast is needed.  R_{L-1} tile 0 (off the per-step chain)
// writes the hypotheses.
//
// Warp roles inside a CTA: warp 0 = TMA producer, warp 1 = MMA issuer
// (elect.sync inside a converged warp: issuing from a divergent lane costs
// 3-4x, scripts/mb_tc.cu), warps 2-17 = epilogue + replicated control.
#pragma once

#include <cuda_fp16.h>

#include "common.cuh"

namespace rnntg {
namespace ptc {

#ifndef NEPI_CFG
#define NEPI_CFG 512  // A/B after the footprint cuts: 16 warps x 8 rows -0.07 (C2) .. -0.13 (C4) us/step vs 8 x 16
#endif
constexpr int NEPI = NEPI_CFG;   // epilogue threads: WPQ warps per TMEM lane quadrant
constexpr int NTH = 64 + NEPI;
constexpr int WPQ = NEPI / 128;  // 2 (default) or 4
constexpr int NR = 32 / WPQ;     // batch rows per epilogue thread (16 or 8)
constexpr int LOG_NR = NR == 16 ? 4 : 3;
static_assert(NEPI == 256 || NEPI == 512, "epilogue: 8 or 16 warps");
#ifndef NSTAGE_CFG
#define NSTAGE_CFG 4
#endif
constexpr int NSTAGE = NSTAGE_CFG;
#ifndef MAXNJ_CFG
#define MAXNJ_CFG 16
#endif
constexpr int MAXNJ = MAXNJ_CFG;       // joint tiles (V+1+D <= 2048)
constexpr int CHUNK = 8192;      // [64 rows][64 k] fp16, SWIZZLE_128B
constexpr int MAXB = 32;         // rows per group (one MMA N slice: 32 hi + 32 lo activation rows)
constexpr int MAXG = 8;          // row groups per kernel: batch <= 256
constexpr int MAXI = 2;          // instances per kernel
constexpr int NSV = 16;          // per-thread state floats saved per group (P: gp; cells: c, h; R_0: + hh0)
constexpr int MAXKP = 640;       // K <= 640: W_lo (K/2 TMEM columns) + 2 x 96 accumulator columns
constexpr int MAXKC = MAXKP / 64;
constexpr int TRUNK = MAXL;      // activation buffer ids: h_0..h_{L-1}, trunk
constexpr int MAXBUF = MAXL + 1;
#ifndef NSLOT_CFG
#define NSLOT_CFG 8  // A/B at -O1: 8 slots -0.22 (C2) / -0.09 (C3) / -0.08 (C4) us/step vs 16
#endif
constexpr int NSLOT = NSLOT_CFG;  // joint-partial ring depth (ack checked every NSLOT/2 steps)
constexpr int CSTRIDE = 32;      // u32 words between counters (one 128-byte line each)

// (ROLE_E, a weightless emitter CTA, and I_0, a weightless layer-0 cell, are
// no longer assigned: J tile 0 emits, R_0 runs the layer-0 cell)
enum Role { ROLE_J = 0, ROLE_P = 1, ROLE_R = 2, ROLE_I = 3, ROLE_E = 4 };  // E: emitter (no weights)
constexpr int NROLES = 5;
#ifndef TANH_SIG
#define TANH_SIG 1
#endif
// Weight operand layout (per CTA, K = KC chunks of 64):
//  - W_hi (fp16 pairs) in TMEM from column WLO_COL, chunk kc at WLO_COL + 32 kc;
//    the product A_hi x [x_hi | x_lo] is a TS MMA with N = 64 into D1;
//  - W_lo of the first nlo_chunks(KC) chunks in TMEM too (after W_hi), the rest
//    as a SWIZZLE_128B smem image; A_lo x x_hi is TS (TMEM) or SS (smem), N = 32,
//    into its own 32 columns D2.
// One 96-column accumulator set [D1 (64) | D2 (32)] leaves 416 columns for
// weights.  Measured per 16-deep k-step (scripts/mb_mma.cu, mb_pipe2.cu): TS+SS
// ~78 cycles (SS is smem-read bound), TS+TS ~52; in the executor the TMEM-W_lo
// chunks run ~280 cycles against ~340 (A/B -0.23 us/step).  A per-chunk runtime
// branch between the two forms inside the unrolled loop cost ~2 us/step, so the
// MMA warp dispatches once per round to a body templated on the chunk count.
constexpr bool SWAP_HILO = true;  // W_hi in TMEM, W_lo (mostly) in smem: the packing convention
#ifndef ACC64
#define ACC64 1  // W_lo.A_hi accumulates into the A_hi columns of W_hi.[A_hi | A_lo]: 64-column accumulator
#endif
constexpr int ACC_COLS = ACC64 ? 64 : 96;  // [hi.x_hi (+ lo.x_hi) | hi.x_lo] (| lo.x_hi)
constexpr int NACC = 1;           // accumulator sets (two measured 0.05 us/step slower)
constexpr int WLO_COL = NACC * ACC_COLS;  // first TMEM weight column
constexpr int MAXNLO = (512 - WLO_COL) / 32 / 2;  // 7 (ACC64) / 6: bound of nlo_chunks over KC
static_assert(MAXNLO <= 7, "mma_round dispatch covers nlo 0..6 and MAXNLO");
#ifndef NLO_MAX
#define NLO_MAX MAXNLO  // A/B knob: cap on the TMEM-resident W_lo chunks
#endif
// chunks whose W_lo is TMEM-resident too (after the KC chunks of W_hi pairs)
__host__ __device__ constexpr int nlo_chunks(int KC) {
  return ((512 - WLO_COL) / 32 - KC < KC ? (512 - WLO_COL) / 32 - KC : KC) < NLO_MAX
             ? ((512 - WLO_COL) / 32 - KC < KC ? (512 - WLO_COL) / 32 - KC : KC)
             : NLO_MAX;
}
// The event trace (RNNTG_PROF) lives in a separate instantiation of the kernel
// (template flag TR): compiled into the product kernel, its runtime-gated code
// cost 0.42 us/step at C2 (~3400 of ~24200 SASS instructions; A/B)
#define PPROF(X) (TR ? (X).prof : (unsigned long long*)nullptr)
#define PECHO(X) (TR ? (X).echo : (unsigned long long*)nullptr)

// counter word indices (times CSTRIDE)
__host__ __device__ inline int cidx_act(int buf, int kc) { return buf * MAXKC + kc; }
__host__ __device__ inline int cidx_hh(int l, int t) { return MAXBUF * MAXKC + l * 64 + t; }
__host__ __device__ inline int cidx_part() { return MAXBUF * MAXKC + MAXL * 64; }
constexpr int NCOUNTERS = MAXBUF * MAXKC + MAXL * 64 + 1;  // per group

struct TParams {
  // Activation buffer b is a 2-D fp16 tensor [ngrp x 2 parity x 64 rows][Kp]
  // (row-major; group g parity e at rows 64 (2g + e) .. +63: 32 hi rows, 32 lo
  // rows); ldmap: box 64 x 64, SWIZZLE_128B (lands in UMMA canonical layout);
  // stmap: the producers' box (32 x 64 plain for LSTM tiles, 64 x 64
  // SWIZZLE_128B from canonical staging otherwise)
  CUtensorMap ldmap[MAXBUF];
  CUtensorMap stmap[MAXBUF];
  int G, B, T, ms, cap, algo, L, cell;
  int H, Hp, J, Jp, V1, D;
  int NJ;                     // joint tiles
  int GH, Gg;                 // table0 row stride / gates per unit
  int ngrp;                   // row groups (<= MAXB rows each), decoded interleaved by every CTA
  int gr0[MAXG + 1];          // group g = batch rows [gr0[g], gr0[g + 1])
  long long max_iters;
  int durations[MAXD];
  const int4* roles;          // [G] {role, layer, tile, float bits of 2^-s}
  const unsigned char* wimg;  // [G][wstride]: W_hi smem image, then W_lo packed [Kp/2][128] u32
  size_t wstride;
  size_t wtoff;               // byte offset of the TMEM column-pair image in a CTA's weight image
  const float* bias[MAXL];    // reference layout [G*H]
  const float* table0;        // [V1][GH] gate-interleaved (col = u*Gg + g)
  const float* fp;            // [B*T][Jp] encoder projection (K1)
  const int* out_len;
  unsigned char* act[MAXBUF];  // [ngrp][2 parity][64 rows][Kp] fp16
  int act_kc[MAXBUF];
  int nprod[MAXBUF][MAXKC];   // producers per chunk
  float* hh[MAXL];            // [ngrp][2 parity][tiles][32 rows][128]: h_l @ W_hh_l from R_l
  unsigned long long* pw;     // [ngrp][NSLOT][2][NJ][32] argmax words {best f32 | idx << 8 | tag}, vocab / duration
  float2* ps;                 // [ngrp][NSLOT][NJ][32] vocab (row max, sumexp) for the emitted score
  unsigned* cnt;              // [ngrp][NCOUNTERS * CSTRIDE]
  unsigned* ack;              // [ngrp][G] per-CTA ack words: steps whose argmax words / partials the CTA consumed
  float* gst;                 // [ngrp][G][NSV][NEPI] per-thread epilogue state of the groups not in flight
  int* tokens;
  int* frames;
  float* scores;
  int* durs;
  int* counts;
  Ctrl* ctrl;
  unsigned long long* prof;   // optional event trace [NEV][PROF_WIN] (first CTA of each role)
  int prof_first[NROLES];     // first CTA index per role (tracing CTAs)
  // step launches (the CUDA-graph executor's loop body and the host loop):
  // STEP_NONE = the whole decode in one launch; STEP_INIT = P0 of every group;
  // STEP_ONE = one decision of every live group, then the loop flags
  int step_mode;
  int* ctl;                   // [G][CTL_INTS] each CTA's replicated control state between step launches
  cudaGraphConditionalHandle h_outer, h_inner;
  int use_cond;               // set the conditional handles (graph bodies)
  int steps_per_launch;       // STEP_ONE: decisions per live group per launch (the loop body unrolled)
  int pdl;                    // step launches as programmatic dependents: weights before griddepcontrol.wait
  int split0;                 // 1: layer-0 cell on its own CTAs (I_0) + an emitter CTA (E); 0: merged into R_0
  // instances: independent CTA sets, each decoding its own row groups
  // (roles[c].y >> 8 = instance); groups [ig0[i], ig0[i+1]), CTAs [ic0[i], ic0[i+1])
  int ninst;
  int ig0[MAXI + 1];
  int ic0[MAXI + 1];
  unsigned long long* stamps;  // optional [G][16] globaltimer stamps of the last launch (RNNTG_STAMPS)
  float* dbg_logits;          // optional [B][V1 + D]: the J tiles' fp32 logits of decision step dbg_step
  int dbg_step;               // (logit-level parity of the tensor-core executor, rnntg_debug_logits)
};
#ifndef STAMPS
#define STAMPS 0  // compile the RNNTG_STAMPS launch stamps in (A/B builds: the checks cost in the hot loop)
#endif
// stamps[slot][cta][16], slot = (group 0's step at launch start) % 64
__device__ __forceinline__ void stamp_at(const TParams& P, int slot, int i, unsigned long long t) {
  if (STAMPS && P.stamps) P.stamps[((size_t)(slot & 63) * P.G + blockIdx.x) * 16 + i] = t;
}
__device__ __forceinline__ void stamp(const TParams& P, int slot, int i) {
  if (STAMPS && P.stamps) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    stamp_at(P, slot, i, t);
  }
}
enum { STEP_NONE = 0, STEP_INIT = 1, STEP_ONE = 2 };
constexpr int PROF_WIN = 64;  // traced joint steps [PROF_S0, PROF_S0 + PROF_WIN)
constexpr int PROF_S0 = 100;
constexpr int NEV = 136;  // 40..47: globaltimer hand-off marks; 48..53: I1/P load + MMA marks;
                          // 56..90 J / 92..126 I1 per-chunk clock64 (load issue, full, issued, acc)

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  // K-major SWIZZLE_128B: 8-row groups 1024 B apart (SBO), LBO unused, sm100 version bit
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  // D f32, A/B f16, both K-major
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// One 64-deep chunk (4 k-steps of K = 16) under ONE elect.sync, then the
// stage commit: D1[0:64) += A_hi x B (TMEM A, N = 64) and D2[0:32) +=
// A_lo x B[:, 0:32) with A_lo from a smem descriptor (ts2) or TMEM (tt2).
// A per-MMA elect block cost ~10 SASS instructions of ELECT/VOTE/R2UR each
// and the MMA warp's issue rate paced the phases (A/B -0.23 us/step).  first:
// the chunk starts the tile (its MMAs overwrite D1 / D2).
__device__ __forceinline__ void mma_chunk_ts2(uint32_t d1, uint32_t d2, uint32_t ahi, uint64_t alo, uint64_t b,
                                              uint32_t first, uint32_t id64, uint32_t id32, uint64_t* bar,
                                              uint32_t first2) {
  asm volatile(
      "{\n\t.reg .pred p, q, t, e;\n\t.reg .b32 h1, h2, h3;\n\t.reg .b64 l1, l2, l3, b1, b2, b3;\n\t"
      "setp.eq.b32 p, %5, 0;\n\tsetp.eq.b32 q, %9, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
      "add.u32 h1, %2, 8;\n\tadd.u32 h2, %2, 16;\n\tadd.u32 h3, %2, 24;\n\t"
      "add.u64 l1, %3, 2;\n\tadd.u64 l2, %3, 4;\n\tadd.u64 l3, %3, 6;\n\t"
      "add.u64 b1, %4, 2;\n\tadd.u64 b2, %4, 4;\n\tadd.u64 b3, %4, 6;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %4, %6, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], %3, %4, %7, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h1], b1, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], l1, b1, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h2], b2, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], l2, b2, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h3], b3, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], l3, b3, %7, t;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n\t}" ::"r"(d1),
      "r"(d2), "r"(ahi), "l"(alo), "l"(b), "r"(first), "r"(id64), "r"(id32), "r"(smem_u32(bar)), "r"(first2)
      : "memory");
}
// TS x TS chunk with the W_lo product in its own columns d2 (A_lo from TMEM)
__device__ __forceinline__ void mma_chunk_tt2(uint32_t d1, uint32_t d2, uint32_t ahi, uint32_t alo, uint64_t b,
                                              uint32_t first, uint32_t id64, uint32_t id32, uint64_t* bar,
                                              uint32_t first2) {
  asm volatile(
      "{\n\t.reg .pred p, q, t, e;\n\t.reg .b32 h1, h2, h3, l1, l2, l3;\n\t.reg .b64 b1, b2, b3;\n\t"
      "setp.eq.b32 p, %5, 0;\n\tsetp.eq.b32 q, %9, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
      "add.u32 h1, %2, 8;\n\tadd.u32 h2, %2, 16;\n\tadd.u32 h3, %2, 24;\n\t"
      "add.u32 l1, %3, 8;\n\tadd.u32 l2, %3, 16;\n\tadd.u32 l3, %3, 24;\n\t"
      "add.u64 b1, %4, 2;\n\tadd.u64 b2, %4, 4;\n\tadd.u64 b3, %4, 6;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %4, %6, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], [%3], %4, %7, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h1], b1, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], [l1], b1, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h2], b2, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], [l2], b2, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h3], b3, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], [l3], b3, %7, t;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n\t}" ::"r"(d1),
      "r"(d2), "r"(ahi), "r"(alo), "l"(b), "r"(first), "r"(id64), "r"(id32), "r"(smem_u32(bar)), "r"(first2)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
// NR consecutive accumulator columns of this thread's lane
template <int N>
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, uint32_t (&r)[N]) {
  if constexpr (N == 16) tmem_ld16(taddr, r);
  else tmem_ld8(taddr, r);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Cross-CTA hand-off protocol (PTX memory model, gpu scope).
//  producer: data writes (generic stores, or TMA bulk stores completed with
//            cp.async.bulk.wait_group 0 and ordered into the generic proxy by
//            fence.proxy.async.global) -> release pattern (fence.acq_rel.gpu or
//            red.release.gpu) -> counter add;
//  consumer: relaxed spin on the counter (an acquire LOAD compiles to
//            LDG.STRONG.GPU + CCTL.IVALL and polling with it invalidated the
//            SM's L1 continuously: 60 us/step) -> ONE fence.acq_rel.gpu after the
//            spin exits (strong read + fence = acquire pattern, which
//            synchronizes-with the producer's release) -> fence.proxy.async.global
//            before TMA loads of the data.
// MM_PROD / MM_CONS select the producer / consumer halves (A/B):
//   MM_PROD 0 none (round 1: relied on L2 behaviour outside the model),
//           1 fence.proxy.async.global + fence.acq_rel.gpu + relaxed adds,
//           2 fence.proxy.async.global + red.release.gpu,
//           3 fence.acq_rel.gpu only,
//           4 fence.proxy.async.global + fence.release.gpu + relaxed adds
//             (MEMBAR.ALL.GPU alone; acq_rel adds ERRBAR, CGAERRBAR, CCTL.IVALL);
//   MM_CONS 0 none, 1 relaxed spin + fence.acq_rel.gpu,
//           2 acquire polls, 3 relaxed spin + one ld.acquire re-read,
//           4 relaxed spin + fence.acquire.gpu (CCTL.IVALL alone: no second L2 round trip).
#ifndef MM_PROD
#define MM_PROD 4
#endif
#ifndef MM_CONS
#define MM_CONS 4
#endif
// one counter poll (the consumer's strong read)
__device__ __forceinline__ unsigned ld_poll_cnt(const unsigned* p) {
  unsigned v;
  if (MM_CONS == 2) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// after a successful relaxed poll of p
__device__ __forceinline__ void acquire_after(const unsigned* p) {
  if (MM_CONS == 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  if (MM_CONS == 4) asm volatile("fence.acquire.gpu;" ::: "memory");
  if (MM_CONS == 3) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    (void)v;
  }
}
__device__ __forceinline__ void spin_geq(const unsigned* p, unsigned target) {
  while (ld_poll_cnt(p) < target) {
  }
  acquire_after(p);
}
// release pattern: fence.release.gpu (MEMBAR.ALL.GPU) + relaxed add; red.release
// compiles to MEMBAR + ERRBAR + CGAERRBAR + RED
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  if (MM_PROD == 4) {
    asm volatile("fence.release.gpu;" ::: "memory");
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  } else {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  }
}
__device__ __forceinline__ void fence_proxy_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Named barrier / OR-reduction over the epilogue warps.
__device__ __forceinline__ void epi_sync() { asm volatile("barrier.cta.sync.aligned 1, %0;" ::"n"(NEPI) : "memory"); }
__device__ __forceinline__ int epi_or(int v) {
  int r;
  asm volatile(
      "{\n\t.reg .pred q, p;\n\tsetp.ne.s32 q, %1, 0;\n\t"
      "barrier.cta.red.or.aligned.pred p, 1, %2, q;\n\tselp.s32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"(v), "n"(NEPI)
      : "memory");
  return r;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Self-validating argmax word: 8-byte single-copy-atomic {value, idx << 8 | tag}.
// Readers spin on the words themselves (no counter, no release round trip).
__device__ __forceinline__ unsigned step_tag(long long s) { return (unsigned)(s % 255) + 1u; }
__device__ __forceinline__ unsigned long long pack_arg(float v, int idx, unsigned tag) {
  return (unsigned long long)__float_as_uint(v) | ((unsigned long long)(((unsigned)idx << 8) | tag) << 32);
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
#ifndef POLL_LD
#define POLL_LD "ld.relaxed.gpu.global.u64"
#endif
__device__ __forceinline__ unsigned long long ld_poll_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile(POLL_LD " %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_ld2(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_ld2_u(uint32_t dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void tma_st2(const CUtensorMap* map, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(x),
               "r"(y), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_all() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void red_relaxed_add(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// after bulk_commit_wait_all(): the completed bulk-store writes, ordered into
// the generic proxy, then released at gpu scope before the counter adds
__device__ __forceinline__ void release_after_bulk() {
  if (MM_PROD == 1 || MM_PROD == 2 || MM_PROD == 4) asm volatile("fence.proxy.async.global;" ::: "memory");
  if (MM_PROD == 1 || MM_PROD == 3) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  if (MM_PROD == 4) asm volatile("fence.release.gpu;" ::: "memory");
}
#ifndef XP_NOREL
#define XP_NOREL 0  // timing experiments only (unsound; with -DMM_CONS=0): no release fence on the activation publishes
#endif
#ifndef PUB_DIRECT
#define PUB_DIRECT 1  // activation hand-offs: plain stores + release (0: TMA store + wait_group + release)
#endif
#ifndef PUB_ET
#define PUB_ET 0  // epilogue thread that issues the activation bulk stores + publish
#endif
// the counter add that publishes (after release_after_bulk)
__device__ __forceinline__ void publish_add(unsigned* p) {
  if (MM_PROD == 2) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
  else asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void st_relaxed_u32(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// byte offset of (row r, k) inside a [rows x 64] fp16 K-major SWIZZLE_128B chunk
__host__ __device__ inline uint32_t swz(int r, int k) {
  return (uint32_t)(r * 128 + ((((k * 2) >> 4) ^ (r & 7)) << 4) + ((k * 2) & 15));
}

// v -> (hi, lo) fp16 at (row r | 32 + r, k) of a chunk
__device__ __forceinline__ void store_split(unsigned char* chunk, int r, int k, float v) {
  const __half hi = __float2half_rn(v);
  const __half lo = __float2half_rn(v - __half2float(hi));
  *reinterpret_cast<__half*>(chunk + swz(r, k)) = hi;
  *reinterpret_cast<__half*>(chunk + swz(32 + r, k)) = lo;
}

// ------------------------------------------------------------------ smem
struct Smem {
  unsigned char* whi;   // [KC][16384]
  unsigned char* ring;  // [NSTAGE][CHUNK]
  float* xs;            // [4][32][32] gate exchange / [128][33] joint transpose / partial staging
  float4* red;          // [2][8][32] joint column-group partials
  int* label;           // [MAXG][32] replicated row state of every group
  int* flag;            // [MAXG][32] bit0 done (FS) / inactive (LL), bit1 accepted this step
  int* tb;              // [MAXG][32] label-looping cursor t
  int* ub;              // [MAXG][32] label-looping symbols at t
  int* cnt;             // [MAXG][32] emissions
  int* kdec;            // [32] this step's decision (labels, scores, durations)
  float* vdec;
  int* ddec;
  int* misc;            // [0..1] round epochs, [5] decision outcome, [6..7] round groups, [8..13] trace
  int* grp;             // [GS_N][MAXG] per-group scalars (GS_*)
  uint64_t* full;       // [NSTAGE]
  uint64_t* empty;      // [NSTAGE]
  uint64_t* accf;       // [2]
  uint64_t* acce;       // [2]
  uint64_t* cmd;        // [1]
  uint64_t* wbar;       // [1] W_lo (smem image) landed
  uint64_t* wready;     // [1] every epilogue warp's share of the TMEM weights stored
  uint32_t* tslot;
  unsigned long long* dbg;  // [64] per-chunk trace stamps (RNNTG_PROF)
};
enum { LD_INIT = 0, LD_VISIT, LD_MULTI };  // Epi::run's load modes
// per-group scalars: FS frame t, FS symbols at t, step s, prediction epoch p, max(out_len), running
enum { GS_T = 0, GS_SYM, GS_STEP, GS_PE, GS_MAXLEN, GS_RUN, GS_N };
constexpr int SM_INTS = 5 * MAXG * 32 + 3 * 32 + 16 + GS_N * MAXG;  // 1440: 8-byte aligned end
// a CTA's control state between step launches: the per-group row state and
// scalars, then joint_evals / pred_steps / outer_iters (2 ints each), err
constexpr int CTL_ROWS = 5 * MAXG * 32, CTL_INTS = CTL_ROWS + GS_N * MAXG + 8;

constexpr int XS_FLOATS = 128 * 33;   // epilogue exchange: [128 cols][33] / [4 gates][32][32]
constexpr int RED_F4 = 256;           // argmax merge / word staging / sumexp group scratch (4 KB)
__host__ __device__ inline size_t smem_bytes(int KC) {
  return 1024 /*align slack*/ + (size_t)KC * 16384 + (size_t)NSTAGE * CHUNK + XS_FLOATS * 4 +
         RED_F4 * 16 + SM_INTS * 4 + 16 * 8 + 64 + 512;
}

__device__ inline Smem carve(unsigned char* raw, int KC) {
  Smem s;
  // align with pointer arithmetic on the shared-memory pointer itself (an
  // integer round trip would turn every access into a generic LD/ST)
  unsigned char* base = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  s.whi = base;
  s.ring = base + (size_t)KC * 16384;
  s.xs = reinterpret_cast<float*>(s.ring + NSTAGE * CHUNK);
  s.red = reinterpret_cast<float4*>(s.xs + XS_FLOATS);
  int* ip = reinterpret_cast<int*>(s.red + RED_F4);
  s.label = ip;
  s.flag = ip + MAXG * 32;
  s.tb = ip + 2 * MAXG * 32;
  s.ub = ip + 3 * MAXG * 32;
  s.cnt = ip + 4 * MAXG * 32;
  ip += 5 * MAXG * 32;
  s.kdec = ip;
  s.vdec = reinterpret_cast<float*>(ip + 32);
  s.ddec = ip + 64;
  s.misc = ip + 96;  // 16 words
  s.grp = ip + 112;  // GS_N * MAXG words
  static_assert((SM_INTS * 4) % 8 == 0, "mbarriers need 8-byte alignment");
  uint64_t* bp = reinterpret_cast<uint64_t*>(ip + 112 + GS_N * MAXG);
  s.full = bp;
  s.empty = bp + NSTAGE;
  s.accf = bp + 2 * NSTAGE;
  s.acce = s.accf + 2;
  s.cmd = s.acce + 2;
  s.wbar = s.cmd + 1;
  s.wready = s.wbar + 1;
  s.tslot = reinterpret_cast<uint32_t*>(s.wbar + 2);
  s.dbg = reinterpret_cast<unsigned long long*>(s.wbar + 3);
  return s;
}

// Branchless activations (~1e-7 relative): the libm versions carry slow-path
// calls that serialise the 32-row unrolled epilogue loops.
#ifndef SIGM_FTZ
#define SIGM_FTZ 1  // sigmoid from ex2/rcp .approx.ftz: no subnormal fix-ups on the chain
#endif
__device__ __forceinline__ float sigm(float x) {
  if (SIGM_FTZ) {
    float e, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * -1.4426950408889634f));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
    return r;
  }
  return __fdividef(1.0f, 1.0f + __expf(-x));
}
// (an FMA-pipe Newton reciprocal for the gate sigmoids, halving the MUFU ops,
// measured 0.25 us/step slower: the cell is not MUFU-bound)
__device__ __forceinline__ float tanh_fast(float x) {
  const float a = fabsf(x);
  // |x| < 0.5: odd Taylor series to x^13 (truncation < 1e-7 relative)
  const float x2 = x * x;
  float p = 21844.0f / 6081075.0f;
  p = fmaf(p, x2, -1382.0f / 155925.0f);
  p = fmaf(p, x2, 62.0f / 2835.0f);
  p = fmaf(p, x2, -17.0f / 315.0f);
  p = fmaf(p, x2, 2.0f / 15.0f);
  p = fmaf(p, x2, -1.0f / 3.0f);
  const float small = fmaf(p * x2, x, x);
  // |x| >= 0.5: 1 - 2 / (e^{2|x|} + 1)
  const float big = copysignf(1.0f - __fdividef(2.0f, __expf(2.0f * a) + 1.0f), x);
  return a < 0.5f ? small : big;
}


// ------------------------------------------------------------------ epilogue
// Epilogue + replicated control of one CTA (warps 2-9).  Thread et = 0..255;
// tile row m = 32*q + lane is this thread's TMEM lane (q = warp & 3, the
// quadrant a warp may address), and it owns batch rows r0 .. r0+15 of it
// (r0 = 16 * (et >= 128)): the two warps of a quadrant split the rows.
// The product kernels are also specialised on the decode configuration, SPEC =
// 2 * algo + (LSTM cell): the algorithm's rules and the cell compile to
// straight-line code (-0.51 us/step at C2 against runtime flags, A/B: the hot
// path's instruction footprint matters).  SPEC_GENERIC reads them at run time
// (the traced instantiation).
constexpr int SPEC_GENERIC = -1;
__host__ __device__ constexpr int spec_of(int algo, int cell) { return 2 * algo + (cell == 1 ? 1 : 0); }
template <int SPEC>
struct CfgFlags {
  static constexpr bool fs = SPEC / 2 == ALGO_FS, tdt = SPEC / 2 == ALGO_TDT, lstm = (SPEC & 1) != 0;
  __device__ explicit CfgFlags(const TParams&) {}
};
template <>
struct CfgFlags<SPEC_GENERIC> {
  const bool fs, tdt, lstm;
  __device__ explicit CfgFlags(const TParams& P) : fs(P.algo == ALGO_FS), tdt(P.algo == ALGO_TDT), lstm(P.cell == 1) {}
};

// W_hi (and the first W_lo chunks) -> TMEM, each epilogue warp its share of
// its lane quadrant's columns, then an arrival on wready for the MMA warp.
template <int BATCH>
__device__ __forceinline__ void load_tmem_weights(const uint32_t* lo, int KC, uint32_t tq, int et, uint64_t* wready) {
  const int warp = 2 + (et >> 5), lane = et & 31, q = warp & 3, grp = (warp - 2) >> 2;
  const int mm = 32 * q + lane;
  const int ncol = (KC + nlo_chunks(KC)) * 32;  // W_hi pairs, then the TMEM-resident W_lo pairs
  const int cbeg = grp * (ncol / WPQ), cend = (grp + 1) * (ncol / WPQ);
  // BATCH columns' loads in flight per batch (a load + store per 8 columns put
  // one L2 round trip per 8 columns on every step launch's start)
  for (int c0 = cbeg; c0 < cend; c0 += BATCH) {
    uint32_t r[BATCH];
#pragma unroll
    for (int j = 0; j < BATCH; ++j) r[j] = c0 + j < cend ? __ldg(lo + (size_t)(c0 + j) * 128 + mm) : 0u;
#pragma unroll
    for (int j = 0; j < BATCH; j += 8)
      if (c0 + j < cend) {
        uint32_t r8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) r8[i] = r[j + i];
        tmem_st8(tq + WLO_COL + c0 + j, r8);
      }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(wready);
}

template <bool TR, int SPEC>
struct Epi : CfgFlags<SPEC> {
  using CfgFlags<SPEC>::fs;
  using CfgFlags<SPEC>::tdt;
  using CfgFlags<SPEC>::lstm;
  const TParams& P;
  const Smem& sm;
  const uint32_t tq;  // TMEM address of this warp's lane quadrant
  const int et, m, r0, role, layer, tile, inst;
  const float wsc;
  const int blank;
  const bool c0;      // runs the layer-0 cell (table0[label] + hh0 + b): I_0 (split0) or R_0
  const bool r0m;     // R_0 merged with the cell: then h_0 @ W_hh0 -> hh0 of the next prediction in registers
  // the emitter (merges the J partials: scores, hypotheses): R_{L-1} tile 0,
  // a CTA off the per-step chain (J tile 0 for one-layer models)
  const bool is_emitter;
  // step launches, a group's first visit of the launch: its words / partials
  // (J rotated) and hh_l come from earlier launches (ordered by the kernel
  // boundary), so those waits are skipped; later visits in the same launch wait
  bool words_prev = false;
  const bool tracer;  // event-trace CTA (single-group decodes only)
  // ---- the current item's group (set_group) ----
  int g = 0, B = 0, row0 = 0;
  unsigned* cnt = nullptr;  // this group's counters
  int* label = nullptr;
  int* flag = nullptr;
  int* tb = nullptr;
  int* ub = nullptr;
  int* ecnt = nullptr;
  int maxlen = 0, p = 0;
  long long s = 0;
  // ---- CTA-wide ----
  int round = 0, err = 0, acc_any = 0;
  float ih[NR];  // I_0: table0[label] rows gathered during the decision
  long long joint_evals = 0, pred_steps = 0, outer_iters = 0;
  bool finish = false, frame_end = false;
  unsigned long long t_entry = 0;  // kernel entry (globaltimer), for STAMPS builds
  // STAMPS builds: per-phase clock64 sums of thread 0 -- 0 load, 1 J round,
  // 2 decide, 3 pred/idle, 4 save/ack, 5 word wait (in decide), 6 acc wait (read_acc), 7 total
  long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  __device__ __forceinline__ long long clk() const { return STAMPS ? clock64() : 0; }

  __device__ Epi(const TParams& P_, const Smem& sm_, uint32_t tmem, int et_, int q, int role_, int layer_,
                 int tile_, int inst_, float wsc_)
      : CfgFlags<SPEC>(P_), P(P_), sm(sm_), tq(tmem + ((uint32_t)(32 * q) << 16)), et(et_), m(32 * q + (et_ & 31)),
        r0(NR * (et_ >> 7)), role(role_),
        layer(layer_), tile(tile_), inst(inst_), wsc(wsc_), blank(P_.V1 - 1), c0(P_.split0 ? (role_ == ROLE_I && layer_ == 0) : (role_ == ROLE_R && layer_ == 0)),
        r0m(!P_.split0 && role_ == ROLE_R && layer_ == 0),
        is_emitter(P_.split0 ? role_ == ROLE_E
                   : P_.L > 1 ? (role_ == ROLE_R && layer_ == P_.L - 1 && tile_ == 0) : (role_ == ROLE_J && tile_ == 0)),

        tracer(PPROF(P_) && P_.ngrp == 1 && (int)blockIdx.x == P_.prof_first[role_]) {}

  __device__ __forceinline__ int& gsc(int which) const { return sm.grp[which * MAXG + g]; }
  __device__ __forceinline__ void set_group(int g_) {
    g = g_;
    row0 = P.gr0[g];
    B = P.gr0[g + 1] - row0;
    cnt = P.cnt + (size_t)g * NCOUNTERS * CSTRIDE;
    label = sm.label + 32 * g;
    flag = sm.flag + 32 * g;
    tb = sm.tb + 32 * g;
    ub = sm.ub + 32 * g;
    ecnt = sm.cnt + 32 * g;
    s = gsc(GS_STEP);
    p = gsc(GS_PE);
    maxlen = gsc(GS_MAXLEN);
  }
  // (every thread keeps the same copies; thread 0 writes them back)
  __device__ __forceinline__ void save_group() {
    if (et == 0) {
      gsc(GS_STEP) = (int)s;
      gsc(GS_PE) = p;
    }
  }
  // per-thread state of the groups not in flight (global, this CTA's slice)
  __device__ __forceinline__ float* gstate(int i) const {
    return P.gst + (((size_t)g * P.G + blockIdx.x) * NSV + i) * NEPI + et;
  }

  // per-CTA publish time of step s (all CTAs): prof[(NEV + cta) * PROF_WIN + s - PROF_S0]
  __device__ __forceinline__ void mark_pub() {
    if (PPROF(P) && P.ngrp == 1 && et == 0 && s >= PROF_S0 && s < PROF_S0 + PROF_WIN)
      PPROF(P)[(size_t)(NEV + blockIdx.x) * PROF_WIN + (s - PROF_S0)] = gtimer();
  }
  // hand-off marks (globaltimer, cross-CTA): 40 P trunk published, 42 J words
  // stored, 43 I_0 words seen, 44 I_0 h0 published, 46 I1 h1 published
  __device__ __forceinline__ void gmark(int ev) {
    if (tracer && et == 0 && s >= PROF_S0 && s < PROF_S0 + PROF_WIN)
      PPROF(P)[(size_t)ev * PROF_WIN + (s - PROF_S0)] = gtimer();
  }
  // clock64 mark by thread et == 32 (second epilogue warp)
  __device__ __forceinline__ void mark2(int ev) {
    if (tracer && et == 32 && s >= PROF_S0 && s < PROF_S0 + PROF_WIN)
      PPROF(P)[(size_t)(NEV + P.G + ev) * PROF_WIN + (s - PROF_S0)] = clock64();
  }
  // ev < 32: globaltimer (cross-CTA), ev + 32 slot block: clock64 (intra-CTA, exact)
  __device__ __forceinline__ void mark(int ev) {
    if (tracer && et == 0 && s >= PROF_S0 && s < PROF_S0 + PROF_WIN) {
      // globaltimer reads queue behind outstanding loads: only at step start
      if (ev == 0) PPROF(P)[(size_t)ev * PROF_WIN + (s - PROF_S0)] = gtimer();
      PPROF(P)[(size_t)(NEV + P.G + ev) * PROF_WIN + (s - PROF_S0)] = clock64();
    }
  }
  // I1 / P: producer chunk-0 / last-chunk issue and MMA-issued times of this
  // round (stamped in misc[8..13] by warps 0/1) -> events ev0 .. ev0+2
  __device__ __forceinline__ void log_ld(int ev0) {
    if (tracer && et == 0 && s >= PROF_S0 && s < PROF_S0 + PROF_WIN) {
      const volatile unsigned long long* t = reinterpret_cast<const volatile unsigned long long*>(sm.misc + 8);
      for (int k = 0; k < 3; ++k) PPROF(P)[(size_t)(ev0 + k) * PROF_WIN + (s - PROF_S0)] = t[k];
    }
  }
  // J / I1: per-chunk load-issue and full times, MMA-issued and acc-ready
  // (clock64, this SM) -> events ev0 + [0, 10) issue, + [10, 20) full, +20, +21
  __device__ __forceinline__ void log_chunks(int ev0, long long tacc) {
    if (tracer && et == 0 && s >= PROF_S0 && s < PROF_S0 + PROF_WIN) {
      const volatile unsigned long long* t = sm.dbg;
      const int KC = P.act_kc[role == ROLE_J ? TRUNK : layer - 1];
      for (int k = 0; k < KC && k < 10; ++k) {
        PPROF(P)[(size_t)(ev0 + k) * PROF_WIN + (s - PROF_S0)] = t[k];
        PPROF(P)[(size_t)(ev0 + 10 + k) * PROF_WIN + (s - PROF_S0)] = t[16 + k];
      }
      PPROF(P)[(size_t)(ev0 + 20) * PROF_WIN + (s - PROF_S0)] = t[31];
      PPROF(P)[(size_t)(ev0 + 21) * PROF_WIN + (s - PROF_S0)] = (unsigned long long)tacc;
      PPROF(P)[(size_t)(ev0 + 22) * PROF_WIN + (s - PROF_S0)] = t[11] - t[10];  // polls after chunk 0
      PPROF(P)[(size_t)(ev0 + 23) * PROF_WIN + (s - PROF_S0)] = t[12];  // chunk 2: before empty wait
      PPROF(P)[(size_t)(ev0 + 24) * PROF_WIN + (s - PROF_S0)] = t[13];  // chunk 2: after TMA issue
      for (int k = 0; k < KC && k < 10; ++k)  // chunk landed (observer warp)
        PPROF(P)[(size_t)(ev0 + 25 + k) * PROF_WIN + (s - PROF_S0)] = t[32 + k];
    }
  }
  // W_hi (and the first W_lo chunks) -> TMEM, each epilogue warp its share of
  // its lane quadrant's columns, then wready for the MMA warp.  Done lazily
  // before the first round: with step launches a CTA's decision and the
  // weight-free I_0 chain run before the weight traffic (the whole model,
  // every launch) competes for L2.
  bool wloaded = false;
#ifndef WEAGER
#define WEAGER 0  // A/B: step launches load the TMEM weights before their decision
#endif
#ifndef WBATCH
#define WBATCH 16  // loads in flight per epilogue thread (32: register spills in the product kernels)
#endif
  __device__ __forceinline__ void load_weights() {
    wloaded = true;
    const int in_buf = role == ROLE_J ? TRUNK : role == ROLE_P ? P.L - 1 : role == ROLE_R ? layer : max(layer - 1, 0);
    load_tmem_weights<WBATCH>(reinterpret_cast<const uint32_t*>(P.wimg + (size_t)blockIdx.x * P.wstride + P.wtoff),
                      P.act_kc[in_buf], tq, et, sm.wready);
  }
  // one load+MMA round on this CTA's input: group g, epoch e (-1 = exit)
  __device__ __forceinline__ void post(int e) {
    if (et == 0) {
      sm.misc[round & 1] = e;
      sm.misc[6 + (round & 1)] = g;
      mbar_arrive(sm.cmd);
    }
    ++round;
  }
  // accumulator of round r -> v[i] = (W . A)[m][r0 + i] * 2^-s
  __device__ __forceinline__ void read_acc(int r, float (&v)[NR]) {
    if (tracer && (role == ROLE_J || (role == ROLE_I && layer == 1)) && (et >> 5) == NEPI / 32 - 1) {
      // trace only: when each chunk of round r lands (full-barrier phase), seen
      // by an idle epilogue warp rather than the MMA warp
      const int KC = P.act_kc[role == ROLE_J ? TRUNK : layer - 1];
      for (int kc = 0; kc < KC && kc < 10; ++kc) {
        const int st = kc % NSTAGE, uses = (KC - st + NSTAGE - 1) / NSTAGE;
        mbar_wait(&sm.full[st], (uint32_t)(((long long)r * uses + kc / NSTAGE) & 1));
        if ((et & 31) == 0) sm.dbg[32 + kc] = clock64();
      }
    }
    const int set = NACC == 1 ? 0 : (r & 1);
    const long long tw0 = clk();
    mbar_wait(&sm.accf[set], (uint32_t)(NACC == 1 ? (r & 1) : ((r >> 1) & 1)));
    if (STAMPS) ph[6] += clk() - tw0;
    tc_fence_after();
    const uint32_t a = tq + set * ACC_COLS + r0;
    {
      uint32_t x0[NR], x1[NR];
      tmem_ldn(a, x0);
      tmem_ldn(a + 32, x1);
      if (ACC64) {
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < NR; ++i) v[i] = (__uint_as_float(x0[i]) + __uint_as_float(x1[i])) * wsc;
      } else {
        uint32_t x2[NR];
        tmem_ldn(a + 64, x2);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < NR; ++i)
          v[i] = (__uint_as_float(x0[i]) + (__uint_as_float(x1[i]) + __uint_as_float(x2[i]))) * wsc;
      }
    }
    tc_fence_before();
    __syncwarp();
    if ((et & 31) == 0) mbar_arrive(&sm.acce[set]);  // one arrival per epilogue warp
  }
  __device__ __forceinline__ void wait_counter(int ci, unsigned target) {
    if (et == 0) spin_geq(cnt + (size_t)ci * CSTRIDE, target);
    epi_sync();
  }
  // this CTA's global stores -> visible -> counter += n: the barrier orders
  // every thread's stores before thread 0's release (cumulative at gpu scope)
  __device__ __forceinline__ void bump(int ci, int n = 1) {
    epi_sync();
    if (role == ROLE_P) mark(34);
    if (et == 0)
      for (int i = 0; i < n; ++i) red_release_add(cnt + (size_t)(ci + i) * CSTRIDE, 1);
  }

  // Publish activation chunks staged in shared memory (canonical layout) with
  // TMA tensor stores into this group's rows: wait_group 0 completes the
  // writes, then the proxy fence + release (release_after_bulk) and the
  // counter adds.  stage [n][CHUNK] -> chunks kc0 .. kc0+n-1, counters ci..
  __device__ __forceinline__ void publish_chunks(const unsigned char* stage, int n, int ci, int buf, int kc0,
                                                 int par) {
    if (PUB_DIRECT) {
      // plain 16-byte stores from the staged chunks (smem swizzle undone),
      // then the same release + counter adds as the R roles' hh hand-off
      epi_sync();
      const int Kp = P.act_kc[buf] * 64;
      unsigned char* gbase = P.act[buf] + ((size_t)(2 * g + par) * 64 * Kp + 64 * kc0) * 2;
      for (int i = et; i < n * 512; i += NEPI) {
        const int c = i >> 9, r = (i >> 3) & 63, sg = i & 7;
        const uint4 v = *reinterpret_cast<const uint4*>(stage + (size_t)c * CHUNK + r * 128 + ((sg ^ (r & 7)) << 4));
        *reinterpret_cast<uint4*>(gbase + ((size_t)r * Kp + 64 * c + 8 * sg) * 2) = v;
      }
      epi_sync();
      if (et == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (!XP_NOREL) asm volatile("fence.release.gpu;" ::: "memory");
        for (int c = 0; c < n; ++c) red_relaxed_add(cnt + (size_t)(ci + c) * CSTRIDE, 1);
      }
      return;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    epi_sync();
    if (et == PUB_ET) {
      for (int c = 0; c < n; ++c)
        tma_st2(&P.stmap[buf], 64 * (kc0 + c), 64 * (2 * g + par), stage + (size_t)c * CHUNK);
      bulk_commit_wait_all();
      release_after_bulk();
      for (int c = 0; c < n; ++c) publish_add(cnt + (size_t)(ci + c) * CSTRIDE);
    }
  }

  __device__ void init_rows() {
    if (et < 32) {
      label[et] = blank;
      tb[et] = 0;
      ub[et] = 0;
      ecnt[et] = 0;
      const int len = et < B ? __ldg(&P.out_len[row0 + et]) : 0;
      flag[et] = (et < B ? (fs ? (0 >= len) : !(0 < len)) : 1) | 2;  // every row runs P0
      if (is_emitter && et < B) P.counts[row0 + et] = 0;
    }
    maxlen = 0;
    for (int b = 0; b < B; ++b) maxlen = max(maxlen, __ldg(&P.out_len[row0 + b]));
    s = 0;
    p = 0;
    if (et == 0) {
      gsc(GS_T) = 0;
      gsc(GS_SYM) = 0;
      gsc(GS_MAXLEN) = maxlen;
    }
    epi_sync();
  }

  // ---- J: logits of this tile's 128 columns -> per-row argmax words (critical),
  // then the per-row (max, sumexp) partials for the emitted score (off the path)
  __device__ void joint_round() {
    mark(0);
    post((int)s);
    // the slot-reuse check's ack loads go out before the accumulator wait
    // (their L2 round trip overlaps the MMA; evaluated below)
    const bool ack_due = s >= NSLOT / 2 && s % (NSLOT / 2) == 0;
    unsigned ack_mn = 0xffffffffu;
    if (ack_due && et < 32) {
      const unsigned* ack = P.ack + (size_t)g * P.G;
      for (int c = P.ic0[inst] + et; c < P.ic0[inst + 1]; c += 32) ack_mn = min(ack_mn, ld_relaxed(ack + c));
    }
    float v[NR];
    read_acc(round - 1, v);
    mark(1);
    mark(16);
    const long long tacc = PPROF(P) ? clock64() : 0;
    if (P.dbg_logits && s == P.dbg_step) {  // logit-parity dump (tests only)
      const int colv = 128 * tile + m;
      if (colv < P.V1 + P.D)
        for (int i = 0; i < NR; ++i)
          if (r0 + i < B) P.dbg_logits[(size_t)(row0 + r0 + i) * (P.V1 + P.D) + colv] = v[i];
    }
    // slot reuse: steps s .. s + NSLOT/2 - 1 overwrite the slots of steps
    // s - NSLOT .. s - NSLOT/2 - 1, so EVERY CTA (not their sum: an off-path
    // role such as the emitter may lag) must have acked step s - NSLOT/2.
    // Checked once per half window on the per-CTA ack words (min over CTAs).
    if (ack_due) {
      if (et < 32) {
        const unsigned target = (unsigned)(s - NSLOT / 2 + 1);
        const unsigned* ack = P.ack + (size_t)g * P.G;
        while (__reduce_min_sync(0xffffffffu, ack_mn) < target) {
          ack_mn = 0xffffffffu;
          for (int c = P.ic0[inst] + et; c < P.ic0[inst + 1]; c += 32) ack_mn = min(ack_mn, ld_relaxed(ack + c));
        }
      }
      epi_sync();
    }
    const int slot = (int)(s % NSLOT);
    const unsigned tg = step_tag(s);
    const int V1 = P.V1, VD = P.V1 + P.D;
    const int lane = et & 31, q = m >> 5, grp = et >> 7;
    const int col = 128 * tile + m;
    unsigned long long* pwg = P.pw + (size_t)g * NSLOT * 2 * P.NJ * 32;
    // per-row argmax of the tile straight from registers: a warp reduce-scatter
    // (NR rows over 32 lanes), then the 4 lane-quadrant warps of the same rows
    // merge through smem in column order.  Ties keep the lowest column
    // (argmax_last_into, tensor.cpp:283-289).
    float2* rd = reinterpret_cast<float2*>(sm.red);  // [2 seg][WPQ grp][4 q][NR rows]
    const bool has_dur = P.D && 128 * tile + 127 >= V1 && 128 * tile < VD;
#pragma unroll
    for (int seg = 0; seg < 2; ++seg) {
      if (seg == 1 && !has_dur) break;
      const bool valid = seg == 0 ? col < V1 : (col >= V1 && col < VD);
      const int cid = seg == 0 ? col : col - V1;
      float a[NR];
      int ai[NR];
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        a[i] = valid ? v[i] : -INFINITY;
        ai[i] = cid;
      }
      // scatter: lane bit (16 >> st) picks which half of the remaining rows
      // this lane keeps; after LOG_NR stages lane bits 16.. hold the row
#pragma unroll
      for (int st = 0; st < LOG_NR; ++st) {
        const int o = 16 >> st, n = (NR / 2) >> st;
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < n; ++i) {
          float keep = up ? a[n + i] : a[i];
          int keepi = up ? ai[n + i] : ai[i];
          const float send = up ? a[i] : a[n + i];
          const int sendi = up ? ai[i] : ai[n + i];
          const float got = __shfl_xor_sync(0xffffffffu, send, o);
          const int goti = __shfl_xor_sync(0xffffffffu, sendi, o);
          const bool b = got > keep || (got == keep && goti < keepi);
          a[i] = b ? got : keep;
          ai[i] = b ? goti : keepi;
        }
      }
      // the remaining 32 / NR lanes per row hold the same row: plain reduce
#pragma unroll
      for (int o = (16 >> LOG_NR); o >= 1; o >>= 1) {
        const float got = __shfl_xor_sync(0xffffffffu, a[0], o);
        const int goti = __shfl_xor_sync(0xffffffffu, ai[0], o);
        const bool b = got > a[0] || (got == a[0] && goti < ai[0]);
        a[0] = b ? got : a[0];
        ai[0] = b ? goti : ai[0];
      }
      if (!(lane & ((32 / NR) - 1))) {
        int row = 0;
#pragma unroll
        for (int st = 0; st < LOG_NR; ++st) row += ((lane >> (4 - st)) & 1) * ((NR / 2) >> st);
        rd[((seg * WPQ + grp) * 4 + q) * NR + row] = make_float2(a[0], __int_as_float(ai[0]));
      }
    }
    mark(17);
    epi_sync();
    if (et < 64) {  // et < 32: vocab rows, 32..63: duration rows
      const int seg = et >> 5, rr = et & 31, g2 = rr / NR, row = rr % NR;
      if (seg == 0 || has_dur) {
        float bv = -INFINITY;
        int bi = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 t = rd[((seg * WPQ + g2) * 4 + k) * NR + row];
          if (t.x > bv) {  // quadrants in column order: strict > keeps the lowest column
            bv = t.x;
            bi = __float_as_int(t.y);
          }
        }
        // the tagged word goes out straight from the merging thread (no staging
        // barrier); tiles without duration columns publish no duration word
        st_relaxed_u64(pwg + (((size_t)slot * 2 + seg) * P.NJ + tile) * 32 + rr, pack_arg(bv, bi, tg));
        if (seg == 0) sm.vdec[rr] = bv;  // this tile's row max, for the sumexp pass
      }
    }
    mark(18);
    gmark(42);
    mark_pub();
    if (PPROF(P)) log_chunks(56, tacc);  // trace only, after the critical part
    float* xs = sm.xs;  // [128 cols][33]
#pragma unroll
    for (int i = 0; i < NR; ++i) xs[m * 33 + r0 + i] = v[i];
    epi_sync();
    constexpr int NW = NEPI / 32, CPW = 128 / NW;  // epilogue warps, columns per warp
    const int r = et & 31, qq = et >> 5;
    const int cb = 128 * tile + CPW * qq;
    float* redf = reinterpret_cast<float*>(sm.red);  // [NW][32] (rd is done)
    // sumexp over the vocab columns relative to the tile's row max
    {
      const float M = sm.vdec[r];
      float ev = 0.0f;
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const float x = xs[(CPW * qq + c) * 33 + r];
        ev += (cb + c < V1) ? __expf(x - M) : 0.0f;
      }
      redf[qq * 32 + r] = ev;
    }
    epi_sync();
    if (et < 32) {
      float S = 0.0f;
#pragma unroll
      for (int k = 0; k < NW; ++k) S += redf[k * 32 + et];
      P.ps[(((size_t)g * NSLOT + slot) * P.NJ + tile) * 32 + et] = make_float2(sm.vdec[et], S);
    }
    epi_sync();
    if (et == 0) red_release_add(cnt + (size_t)cidx_part() * CSTRIDE, 1);
    mark(2);
  }

  // table0[label] rows of this thread's gate row for the next layer-0 cell
  // (issued early; consumed only in the cell, so the loads stay in flight)
  __device__ __forceinline__ void gather_table0() {
    // (units past Hp exist only in the last tile and are masked in the cell;
    // clamped so the last table row's gather stays inside the table)
    const int unit = min(lstm ? 32 * tile + (m >> 2) : 128 * tile + m, P.Hp - 1), gate = lstm ? (m & 3) : 0;
    // unconditional loads (rows >= B carry the blank label, a valid row): a
    // predicated load compiles to load + select and the warp stalls on it
#pragma unroll
    for (int i = 0; i < NR; ++i)
      ih[i] = __ldg(&P.table0[(size_t)sm.kdec[r0 + i] * P.GH + unit * P.Gg + gate]);
  }

  // ---- replicated decision of step s.  The first epilogue warp (lane = row)
  // spins on the J tiles' tagged argmax words, applies the rules and reduces
  // the row flags with ballots; ONE barrier then publishes the outcome.
  // The emitter also merges the (max, sumexp) partials for the score.
  __device__ void decide() {
    if (c0) gmark(41);
    if (et < 32) {
      const int b = et;
      const bool valid = b < B;
      const int slot = (int)(s % NSLOT);
      const unsigned tg = step_tag(s);
      const bool emitter = is_emitter;
      int kk = blank, dd = 0, npoll_out = 0;
      long long lat1_out = 0;
      float best = 0.0f;
      if (valid) {
        const unsigned long long* wv = P.pw + (size_t)g * NSLOT * 2 * P.NJ * 32 + ((size_t)slot * 2 * P.NJ) * 32 + b;
        const unsigned long long* wd = wv + (size_t)P.NJ * 32;
        unsigned long long a[MAXNJ], d0 = 0ull, d1 = 0ull;
#pragma unroll
        for (int t = 0; t < MAXNJ; ++t) a[t] = 0ull;
        __syncwarp(0xffffffffu >> (32 - B));
        bool ok;
        const int nj = P.NJ;
        const bool hasd = P.D != 0;
        // only the tiles holding duration columns carry duration partials
        const int td0 = P.V1 / 128, td1 = (P.V1 + P.D - 1) / 128;
        int npoll = 0;
        long long lat1 = 0;
        if (tracer && c0 && b == 0) {  // one strong load, timed
          const long long cl0 = clock64();
          const unsigned long long w0 = ld_poll_u64(wv);
          long long cl1 = 0;
          if (w0 != 0x123456789abcdefull) cl1 = clock64();  // the branch waits for the load
          lat1 = cl1 - cl0;
        }
        // spin on one word (tile NJ-1) with a single load in flight, then read
        // the rest once (warp-wide strong loads are serviced ~100 cycles apart:
        // a 9-16 load batch per poll made each poll ~1 us; one load is ~360 cycles)
        const long long tw0 = clk();
        // (step launches: J wrote step s's words in the previous launch)
        if (!words_prev)
          while ((unsigned)(ld_poll_u64(wv + (nj - 1) * 32) >> 32 & 0xffu) != tg) ++npoll;
        if (c0 && b == 0) mark(30);  // last tile's word seen
        do {
          ++npoll;
          ok = true;
          // branch-free: every slot loads (clamped to a valid tile), so all
          // loads are in flight together; a branch per load serialised them
          // (one ~300-cycle round trip each, ~2000 cycles per poll)
#pragma unroll
          for (int t = 0; t < MAXNJ; ++t)
            if (t < nj) a[t] = ld_poll_u64(wv + t * 32);
          if (hasd) {
            d0 = ld_poll_u64(wd + td0 * 32);
            d1 = ld_poll_u64(wd + td1 * 32);
          }
          // branch-free tag check: a short-circuit && compiled to one branch +
          // reconvergence block per tile (~1000 cycles for 16 tiles)
          unsigned bad = (unsigned)hasd & ((unsigned)((((unsigned)(d0 >> 32)) & 0xffu) != tg) |
                                           (unsigned)((((unsigned)(d1 >> 32)) & 0xffu) != tg));
#pragma unroll
          for (int t = 0; t < MAXNJ; ++t) {
            const unsigned ta = (unsigned)(a[t] >> 32) & 0xffu;
            bad |= (unsigned)(t < nj) & (unsigned)(ta != tg);
          }
          ok = bad == 0u;
        } while (!ok);
        if (c0 && b == 0) mark(31);  // every tile's word seen
        if (STAMPS) ph[5] += clk() - tw0;
        npoll_out = npoll;
        lat1_out = lat1;
        best = -INFINITY;
        // selects, no branches; tiles in column order: strict > keeps the lowest
        // index (a 4-level tree merge measured 0.2 us/step slower)
#pragma unroll
        for (int t = 0; t < MAXNJ; ++t) {
          const float x = __uint_as_float((unsigned)a[t]);
          const bool tx = (t < nj) & (x > best);
          best = tx ? x : best;
          kk = tx ? (int)((unsigned)(a[t] >> 32) >> 8) : kk;
        }
        // durations: tile td0 first (column order), td1 only if strictly greater
        int di = (int)((unsigned)(d0 >> 32) >> 8);
        if (__uint_as_float((unsigned)d1) > __uint_as_float((unsigned)d0)) di = (int)((unsigned)(d1 >> 32) >> 8);
        dd = hasd ? P.durations[di] : 0;
      }
      sm.kdec[b] = kk;
      if (c0 && tracer && b == 0 && s >= PROF_S0 && s < PROF_S0 + PROF_WIN)
        PPROF(P)[(size_t)39 * PROF_WIN + (s - PROF_S0)] = (unsigned long long)npoll_out,
        PPROF(P)[(size_t)38 * PROF_WIN + (s - PROF_S0)] = (unsigned long long)lat1_out;
      if (c0) {
        // hand the labels to the other epilogue warps now: their table0
        // gathers for the layer-0 cell overlap the rules below; this warp's
        // own gather (rows r0.., labels of lanes r0..) goes out first too
        __syncwarp();
        asm volatile("barrier.cta.arrive.aligned 2, %0;" ::"n"(NEPI) : "memory");
        gather_table0();
        mark(22);
        gmark(43);
      }
      float v = 0.0f;
      if (emitter) {
        if (b == 0 && !words_prev) spin_geq(cnt + (size_t)cidx_part() * CSTRIDE, (unsigned)P.NJ * (unsigned)(s + 1));
        __syncwarp();
        if (valid) {
          float Mx = -INFINITY, Sx = 0.0f;
          const float2* psg = P.ps + ((size_t)g * NSLOT + slot) * P.NJ * 32;
          for (int t = 0; t < P.NJ; ++t) {
            const float2 pv = __ldcg(&psg[(size_t)t * 32 + b]);
            if (pv.x != -INFINITY) {
              const float nm = fmaxf(Mx, pv.x);
              Sx = (Sx == 0.0f ? 0.0f : Sx * __expf(Mx - nm)) + pv.y * __expf(pv.x - nm);
              Mx = nm;
            }
          }
          v = best - (Mx + logf(Sx));  // logp of the argmax (log_softmax_into, tensor.cpp:463-480)
        }
      }
      // decision rules, lane per row (decoders.cpp:261-307 / 432-512)
      const int t_fs = gsc(GS_T);
      int f = flag[b] & ~2;
      if (valid) {
        const int k = kk;
        const int rg = row0 + b;  // batch row
        if (fs) {
          if (!(f & 1)) {
            if (k == blank) {
              f |= 1;
            } else {
              const int nb = ecnt[b];
              if (emitter && nb < P.cap) {
                const size_t o = (size_t)rg * P.cap + nb;
                P.tokens[o] = k;
                P.frames[o] = t_fs;
                P.scores[o] = v;
                P.durs[o] = 0;
                P.counts[rg] = nb + 1;
              }
              ecnt[b] = nb + 1;
              label[b] = k;
              f |= 2;
            }
          }
        } else if (!(f & 1)) {
          const int len = __ldg(&P.out_len[rg]);
          int t = tb[b], u = ub[b];
          if (k == blank) {
            const int d = tdt ? dd : 1;
            t += d > 1 ? d : 1;
            u = 0;
          } else {
            const int d = tdt ? dd : 0;
            const int nb = ecnt[b];
            if (emitter && nb < P.cap) {
              const size_t o = (size_t)rg * P.cap + nb;
              P.tokens[o] = k;
              P.frames[o] = t;
              P.scores[o] = v;
              P.durs[o] = d;
              P.counts[rg] = nb + 1;
            }
            ecnt[b] = nb + 1;
            label[b] = k;
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
          tb[b] = t;
          ub[b] = u;
          if (!(t < len)) f |= 1;
        }
      }
      const bool acc_b = valid && ((f >> 1) & 1), live_b = valid && !(f & 1);
      const bool accany = __ballot_sync(0xffffffffu, acc_b) != 0;
      const bool liveany = __ballot_sync(0xffffffffu, live_b) != 0;
      bool fin = false, frame_end = false;
      if (fs) {
        int sym = gsc(GS_SYM) + 1;
        int t = t_fs;
        if (!liveany || sym >= P.ms) {  // frame ends (decoders.cpp:297-313)
          frame_end = true;
          t += 1;
          sym = 0;
          if (t >= maxlen) fin = true;
          if (valid) f = (f & 2) | (t >= __ldg(&P.out_len[row0 + b]) ? 1 : 0);
        }
        __syncwarp();
        if (b == 0) {
          gsc(GS_SYM) = sym;
          gsc(GS_T) = t;
        }
      } else {
        fin = !liveany;
      }
      if (s + 1 > P.max_iters) fin = true;  // runaway cap (engine.cpp:286-290), per group
      flag[b] = f;
      if (b == 0) sm.misc[5] = (accany ? 1 : 0) | (fin ? 2 : 0) | (frame_end ? 4 : 0);
      if (c0) mark(24);
    } else if (c0) {
      asm volatile("barrier.cta.sync.aligned 2, %0;" ::"n"(NEPI) : "memory");
      mark2(35);
      gather_table0();
      mark2(36);
    }
    epi_sync();
    if (c0) mark2(37);
    const int o = sm.misc[5];
    acc_any = o & 1;
    finish = (o >> 1) & 1;
    frame_end = (o >> 2) & 1;
    if (o & 4) ++outer_iters;
    ++joint_evals;
    if (s + 1 > P.max_iters) err = ERR_RUNAWAY;
    mark(role == ROLE_J ? 3 : role == ROLE_R ? 10 : c0 ? 4 : role == ROLE_I ? 6 : role == ROLE_E ? 15 : 8);
  }

  // ---- the decode skeleton.  Every group starts with P0 = pred(blank, 0)
  // (decoders.cpp:414-430); then the live groups are visited round-robin, one
  // decision per visit: pred(te) after an accepting decision, idle(te)
  // otherwise.  load(mode) starts every visit: mode LD_INIT before a group's
  // P0 (the role's per-thread state of the group := zero), LD_VISIT with one
  // group, LD_MULTI with several (the state of the visited group moves from
  // global memory into registers first); save() moves it back (several
  // groups only).
  // the next live group of this instance after the current one (round-robin order)
  __device__ __forceinline__ int next_live() const {
    const int n = P.ig0[inst + 1] - P.ig0[inst];
    for (int k = 1; k <= n; ++k) {
      const int gg = P.ig0[inst] + (g - P.ig0[inst] + k) % n;
      if (sm.grp[GS_RUN * MAXG + gg]) return gg;
    }
    return g;
  }
  // lag: with several live groups, P and the pure R roles leave their MMA
  // running and finish the previous group's epilogue on their next visit,
  // after its decision (fin), so the visit does not span the upstream chain
  // (not in the P0 pass: no visit in between would finish the lagged epilogue)
  bool in_init = false;
  __device__ __forceinline__ bool lag_ok() const { return P.step_mode == STEP_NONE && !in_init && next_live() != g; }

  template <typename Pred, typename Idle, typename Load, typename Save, typename Fin>
  __device__ void run(Pred&& pred, Idle&& idle, Load&& load, Save&& save, Fin&& fin) {
    const int mode = P.step_mode;
    // with several groups or step launches, the per-thread state of a group
    // lives in global memory between its visits
    const bool multi = P.ngrp > 1 || mode != STEP_NONE;
    ph[7] = clk();
    int sslot = 0;
    // the TMEM weights before the first round: at the start of a whole-decode
    // or P0 launch; in a step launch after its first decision (the decision
    // and R_0's weight-free layer-0 cell go first, before the weight traffic),
    // except I_1, the first MMA after the decision, which loads before it
    const bool has_w = role != ROLE_E && !(role == ROLE_I && layer == 0);
    if (has_w && (WEAGER || P.pdl || (role == ROLE_I && layer == 1) || (role == ROLE_R && layer == 0 && !r0m)))
      load_weights();
    // a programmatic-dependent step launch started while the previous one was
    // finishing: everything above only touched the weights; the decode state
    // (control blocks, counters, words, activations) after the primary grid
    if (P.pdl) pdl_wait();
    if (mode != STEP_ONE) {  // (shared memory is not zeroed at launch: no stale running flags)
      for (int i = et; i < GS_N * MAXG; i += NEPI) sm.grp[i] = 0;
      epi_sync();
    }
    if (mode == STEP_ONE) {
      load_ctl();
      sslot = sm.grp[GS_STEP * MAXG];
      if (et == 0) {
        stamp_at(P, sslot, 0, t_entry);
        stamp(P, sslot, 2);
      }
    } else {
      if (has_w && !wloaded) load_weights();
      in_init = true;
      for (int gg = P.ig0[inst]; gg < P.ig0[inst + 1]; ++gg) {
        set_group(gg);
        init_rows();
        load(LD_INIT);
        pred(0LL);
        ++pred_steps;
        int live = et < B ? !(flag[et] & 1) : 0;
        live = epi_or(live);
        const bool running0 = fs ? (maxlen > 0) : (live != 0);
        if (et < 32) flag[et] &= ~2;
        if (et == 0) gsc(GS_RUN) = running0 ? 1 : 0;
        if (multi) save();
        if (role == ROLE_J && mode == STEP_INIT && running0) joint_round();  // step 0's joint
        save_group();
        epi_sync();
      }
      in_init = false;
    }
    bool acc_round = false, fend_round = false;
    if (mode != STEP_INIT) {
      for (int rnd = 0;; ++rnd) {
        bool any = false;
        for (int gg = P.ig0[inst]; gg < P.ig0[inst + 1]; ++gg) {
          if (!sm.grp[GS_RUN * MAXG + gg]) continue;
          any = true;
          set_group(gg);
          words_prev = mode == STEP_ONE && rnd == 0;
          if (STAMPS && mode == STEP_NONE) sslot = (int)s;  // whole-decode launches: one slot per step
          long long tp0 = clk();
          load(multi ? LD_MULTI : LD_VISIT);
          if (STAMPS) { const long long t = clk(); ph[0] += t - tp0; tp0 = t; }
          if (et == 0 && gg == 0) stamp(P, sslot, 3);
          if (STAMPS && role == ROLE_J && et == 0 && gg == 0) stamp(P, sslot, 1);  // (J: before its joint)
          // step launches run J at the END of a visit (the next step's joint,
          // so J's weight load overlaps the decision + prediction chain)
          if (role == ROLE_J && mode == STEP_NONE) joint_round();
          if (STAMPS) { const long long t = clk(); ph[1] += t - tp0; tp0 = t; }
          decide();
          fin();  // a lagged epilogue of the previous visit
          if (STAMPS) { const long long t = clk(); ph[2] += t - tp0; tp0 = t; }
          if (has_w && !wloaded && !r0m) load_weights();  // (merged R_0: after its cell, in pred)
          if (et == 0 && gg == 0) stamp(P, sslot, 4);
          fend_round |= frame_end;
          if (finish) {
            if (et == 0) gsc(GS_RUN) = 0;
            epi_sync();
            continue;
          }
          acc_round |= acc_any != 0;
          if (acc_any) {
            ++p;
            pred(s + 1);
            ++pred_steps;
            if (!fs) ++outer_iters;
          } else {
            idle(s + 1);
          }
          if (et == 0 && gg == 0) stamp(P, sslot, 5);
          if (STAMPS) { const long long t = clk(); ph[3] += t - tp0; tp0 = t; }
          if (multi) save();
          // this CTA is done with step s's words: ack (slot reuse, joint_round).
          // A per-CTA word; the reads it covers were consumed before the barrier
          // that precedes it, so it needs no release.
          if (et == 0) st_relaxed_u32(P.ack + (size_t)g * P.G + blockIdx.x, (unsigned)(s + 1));
          ++s;
          if (et < 32) flag[et] &= ~2;
          if (role == ROLE_J && mode == STEP_ONE) joint_round();  // step s + 1's joint
          if (et == 0 && gg == 0) stamp(P, sslot, 6);
          save_group();
          epi_sync();
          if (STAMPS) ph[4] += clk() - tp0;
        }
        if (!any || (mode == STEP_ONE && rnd + 1 >= P.steps_per_launch)) break;
      }
    }
    fin();
    if (STAMPS && mode == STEP_NONE && et == 0) {
      ph[7] = clk() - ph[7];
      for (int i = 0; i < 8; ++i) stamp_at(P, 63, 8 + i, (unsigned long long)ph[i]);
    }
    if (mode != STEP_NONE) {
      // step launches: keep the control state for the next launch, and set
      // the loop flags (frame-looping: the inner WHILE runs a frame's
      // symbols; label-looping: the inner WHILE skips blanks until a row
      // accepts; the outer WHILE runs while any group is live)
      save_ctl();
      if (et == 0) stamp(P, sslot, 7);
      if (blockIdx.x == 0 && et == 0) {
        int run_any = 0;
        for (int gg = 0; gg < P.ngrp; ++gg) run_any |= sm.grp[GS_RUN * MAXG + gg];
        const bool inner = run_any && (fs ? !fend_round : !acc_round);
        P.ctrl->any = run_any;
        P.ctrl->abort = inner ? 1 : 0;  // host loop: the inner loop continues
        if (P.use_cond) {
          cudaGraphSetConditional(P.h_inner, inner ? 1u : 0u);
          cudaGraphSetConditional(P.h_outer, run_any ? 1u : 0u);
        }
      }
    }
  }

  // control state of this CTA <-> its global block (step launches)
  __device__ void load_ctl() {
    const int* c = P.ctl + (size_t)blockIdx.x * CTL_INTS;
    for (int i = et; i < CTL_ROWS; i += NEPI) sm.label[i] = c[i];  // label, flag, tb, ub, cnt: contiguous
    for (int i = et; i < GS_N * MAXG; i += NEPI) sm.grp[i] = c[CTL_ROWS + i];
    const long long* cc = reinterpret_cast<const long long*>(c + CTL_ROWS + GS_N * MAXG);
    joint_evals = cc[0];
    pred_steps = cc[1];
    outer_iters = cc[2];
    err = c[CTL_ROWS + GS_N * MAXG + 6];
    epi_sync();
  }
  __device__ void save_ctl() {
    epi_sync();
    int* c = P.ctl + (size_t)blockIdx.x * CTL_INTS;
    for (int i = et; i < CTL_ROWS; i += NEPI) c[i] = sm.label[i];
    for (int i = et; i < GS_N * MAXG; i += NEPI) c[CTL_ROWS + i] = sm.grp[i];
    if (et == 0) {
      long long* cc = reinterpret_cast<long long*>(c + CTL_ROWS + GS_N * MAXG);
      cc[0] = joint_evals;
      cc[1] = pred_steps;
      cc[2] = outer_iters;
      c[CTL_ROWS + GS_N * MAXG + 6] = err;
    }
  }

  // ---- layer cells: pre-activations (gate row m, rows r0..r0+NR-1) -> committed h.
  // LSTM tiles are unit-major (m = 4*unit + gate): a lane quad holds one unit's
  // i,f,g,o, so the gates meet through a per-warp smem transpose (__syncwarp,
  // no CTA barrier).  Lane (quad qd, slot g') then runs the cell for rows
  // r0 + 4j + g', j < NR / 4.
  __device__ __forceinline__ void cell_lstm(const float (&pre)[NR], int l, int pe, float (&c)[NR / 4],
                                            float (&h)[NR / 4]) {
    const int lane = et & 31, gt = lane & 3, qd = lane >> 2;
    float* xw = sm.xs + (et >> 5) * (NR * 33);  // this warp's [NR rows][33]
    // i, f, o: sigmoid; g: tanh(x) = 2 sigmoid(2x) - 1 (absolute error ~1e-7,
    // what the cell update c' = f c + i g needs; one code path per lane quad)
    const float sc = gt == 2 ? 2.0f : 1.0f;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const float a = sigm(sc * pre[i]);
      xw[i * 33 + lane] = gt == 2 ? 2.0f * a - 1.0f : a;
    }
    __syncwarp();
    const int u = 32 * tile + 8 * (m >> 5) + qd;
    // a tile's 32 units: one 32 x 64 box, staged plain [64 rows][32] fp16
    __half* st16 = reinterpret_cast<__half*>(sm.red);
    const int ul = u - 32 * tile;
    // loads, arithmetic and stores in separate passes: the compiler cannot move
    // a later row's xw loads above an earlier row's st16 stores (both shared
    // memory), which serialised the NR / 4 per-row dependency chains
    float gi[NR / 4], gf[NR / 4], gg[NR / 4], go[NR / 4];
    bool cm[NR / 4];
#pragma unroll
    for (int j = 0; j < NR / 4; ++j) {
      const int i = 4 * j + gt, r = r0 + i;
      gi[j] = xw[i * 33 + 4 * qd];
      gf[j] = xw[i * 33 + 4 * qd + 1];
      gg[j] = xw[i * 33 + 4 * qd + 2];
      go[j] = xw[i * 33 + 4 * qd + 3];
      cm[j] = r < B && (flag[r] & 2);
    }
#pragma unroll
    for (int j = 0; j < NR / 4; ++j) {
      const float cn = gf[j] * c[j] + gi[j] * gg[j];
      // tanh(c) = 2 sigm(2c) - 1 like the g gate (absolute error ~1e-7, what
      // h = o tanh(c) needs): no polynomial branch on the dependency chain
      const float hn = u < P.H ? go[j] * fmaf(2.0f, sigm(2.0f * cn), -1.0f) : 0.0f;
      c[j] = cm[j] ? cn : c[j];
      h[j] = cm[j] ? hn : h[j];
    }
#pragma unroll
    for (int j = 0; j < NR / 4; ++j) {
      const int r = r0 + 4 * j + gt;
      const __half hh = __float2half_rn(h[j]);
      st16[r * 32 + ul] = hh;
      st16[(32 + r) * 32 + ul] = __float2half_rn(h[j] - __half2float(hh));
    }
    __syncwarp();
    if (c0) mark(21);
    if (PUB_DIRECT) {  // see publish_chunks: 256 x 16-byte plain stores, release, counter
      epi_sync();
      const int Kp = P.act_kc[l] * 64;
      if (et < 256) {
        const int r = et >> 2, sg = et & 3;
        const uint4 v = reinterpret_cast<const uint4*>(st16)[et];
        *reinterpret_cast<uint4*>(P.act[l] + (((size_t)(2 * g + (pe & 1)) * 64 + r) * Kp + 32 * tile + 8 * sg) * 2) = v;
      }
      epi_sync();
      if (et == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (!XP_NOREL) asm volatile("fence.release.gpu;" ::: "memory");
        red_relaxed_add(cnt + (size_t)cidx_act(l, (32 * tile) >> 6) * CSTRIDE, 1);
      }
      return;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    epi_sync();
    if (et == PUB_ET) {
      tma_st2(&P.stmap[l], 32 * tile, 64 * (2 * g + (pe & 1)), st16);
      bulk_commit_wait_all();
      release_after_bulk();
      publish_add(cnt + (size_t)cidx_act(l, (32 * tile) >> 6) * CSTRIDE);
    }
  }
  // tanh RNN: one unit per row m (128 units per tile)
  __device__ __forceinline__ void cell_tanh(const float (&pre)[NR], int l, int pe, float (&h)[NR]) {
    const int u = 128 * tile + m;
    unsigned char* stage = reinterpret_cast<unsigned char*>(sm.xs);  // [2][CHUNK] staging
    if (u < P.Hp) {
      unsigned char* ch = stage + (size_t)((u >> 6) & 1) * CHUNK;
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const int r = r0 + i;
        const float hn = u < P.H ? tanh_fast(pre[i]) : 0.0f;
        h[i] = (r < B && (flag[r] & 2)) ? hn : h[i];
        store_split(ch, r, u & 63, h[i]);
      }
    }
    const int cb = (128 * tile) >> 6;
    publish_chunks(stage, min(2, P.act_kc[l] - cb), cidx_act(l, cb), l, cb, pe & 1);
  }

  __device__ void run_role();
};

template <bool TR, int SPEC>
__device__ __forceinline__ void Epi<TR, SPEC>::run_role() {
  const int unit = lstm ? 32 * tile + (m >> 2) : 128 * tile + m;  // LSTM tiles: m = 4*unit + gate
  const int gate = lstm ? (m & 3) : 0;
  auto nop = [&]() {};
  auto nopl = [&](int) {};
  if (role == ROLE_J || role == ROLE_E) {
    run([&](long long) {}, [&](long long) {}, nopl, nop, nop);
  } else if (role == ROLE_P) {
    float gp[NR], fpv[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) gp[i] = 0.0f;
    const int j = 128 * tile + m;
    // fp[b, t_b, j] for the next trunk, t from the latest decision
    auto prefetch = [&]() {
      const int tfs = gsc(GS_T);
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        // unconditional (clamped) loads so the warp does not stall here; rows
        // >= B / columns >= J are masked where the values are used
        const int r = min(r0 + i, B - 1);
        int t = fs ? tfs : tb[r];
        t = t < 0 ? 0 : (t > P.T - 1 ? P.T - 1 : t);
        fpv[i] = __ldg(&P.fp[((size_t)(row0 + r) * P.T + t) * P.Jp + min(j, P.Jp - 1)]);
      }
    };
    auto trunk = [&](long long te, const float (&gpa)[NR]) {  // trunk(te) = relu(fp + gp) -> act[TRUNK]
      mark(32);
      unsigned char* stage = reinterpret_cast<unsigned char*>(sm.xs);  // [2][CHUNK] staging
      if (j < P.Jp) {
        unsigned char* ch = stage + (size_t)((j >> 6) & 1) * CHUNK;
#pragma unroll
        for (int i = 0; i < NR; ++i) {
          const int r = r0 + i;
          const float x = (r < B && j < P.J) ? fmaxf(fpv[i] + gpa[i], 0.0f) : 0.0f;
          store_split(ch, r, j & 63, x);
        }
      }
      const int cb = (128 * tile) >> 6;
      mark(33);
      publish_chunks(stage, min(2, P.act_kc[TRUNK] - cb), cidx_act(TRUNK, cb), TRUNK, cb, (int)(te & 1));
      gmark(40);
    };
    // a lagged pred (several live groups): its trunk finished on the next visit
    int pend_r = -1, pend_g = 0;
    long long pend_te = 0;
    auto finish_pending = [&]() {
      if (pend_r < 0) return;
      const int gcur = g;
      set_group(pend_g);  // (the current group's decision left its s / p untouched)
      float v[NR];
      prefetch();
      read_acc(pend_r, v);
      trunk(pend_te, v);
#pragma unroll
      for (int i = 0; i < NR; ++i) *gstate(i) = v[i];  // the group's gp
      pend_r = -1;
      set_group(gcur);
    };
    run(
        [&](long long te) {
          post(p);
          if (lag_ok()) {
            pend_r = round - 1;
            pend_g = g;
            pend_te = te;
            return;
          }
          prefetch();
          float v[NR];
          read_acc(round - 1, v);
          mark(9);
          log_ld(51);
#pragma unroll
          for (int i = 0; i < NR; ++i) gp[i] = v[i];
          trunk(te, gp);
          mark(14);
          mark_pub();
        },
        [&](long long te) {
          prefetch();
          trunk(te, gp);
        },
        [&](int mode) {
#pragma unroll
          for (int i = 0; i < NR; ++i) gp[i] = mode == LD_MULTI ? *gstate(i) : mode == LD_INIT ? 0.0f : gp[i];
        },
        [&]() {
#pragma unroll
          for (int i = 0; i < NR; ++i) *gstate(i) = gp[i];
        },
        finish_pending);
  } else if (role == ROLE_R && !r0m) {
    // hh_l(p+1) = h_l(p) @ W_hh_l -> global, for the layer-l cell of the next
    // prediction; lagged to the next visit while other groups are live
    int pend_r = -1, pend_g = 0, pend_p = 0;
    auto store_hh = [&](int r, int gq, int pq) {
      float v[NR];
      read_acc(r, v);
      float* hb = P.hh[layer] + ((size_t)(2 * gq + ((pq + 1) & 1)) * 64 + tile) * 32 * 128;
#pragma unroll
      for (int i = 0; i < NR; ++i) hb[(r0 + i) * 128 + m] = v[i];
      epi_sync();  // every thread's stores, then thread 0's release
      if (et == 0) red_release_add(P.cnt + (size_t)gq * NCOUNTERS * CSTRIDE + (size_t)cidx_hh(layer, tile) * CSTRIDE, 1);
    };
    run(
        [&](long long) {
          post(p);
          if (lag_ok()) {
            pend_r = round - 1;
            pend_g = g;
            pend_p = p;
            return;
          }
          store_hh(round - 1, g, p);
          mark_pub();
        },
        [&](long long) {}, nopl, nop,
        [&]() {
          if (pend_r < 0) return;
          store_hh(pend_r, pend_g, pend_p);
          pend_r = -1;
        });
  } else {
    // R_0: the layer-0 cell (table0[label] + hh0 + b), then the next
    // prediction's hh0 = h0 @ W_hh0 into registers (hx); I_l: the W_ih_l MMA
    // plus hh_l from R_l
    const float* bl = P.bias[layer];
    const float bias_m = unit < P.H ? __ldg(&bl[gate * P.H + unit]) : 0.0f;
    float c4[NR / 4], h4[NR / 4], hr[NR], hx[NR];
#pragma unroll
    for (int j = 0; j < NR / 4; ++j) c4[j] = h4[j] = 0.0f;
#pragma unroll
    for (int j = 0; j < NR; ++j) hr[j] = hx[j] = 0.0f;
    // hh_l(pe) (R_l's output, l >= 1) -> x; zero for P0
    auto load_hh = [&](int pe, float (&x)[NR]) {
      if (pe > 0) {
        // (step launches: R_l wrote hh_l(pe) in an earlier launch, ordered by the kernel boundary)
        if (!words_prev) wait_counter(cidx_hh(layer, tile), (unsigned)pe);
        const float* hb = P.hh[layer] + ((size_t)(2 * g + (pe & 1)) * 64 + tile) * 32 * 128;
#pragma unroll
        for (int i = 0; i < NR; ++i) x[i] = __ldcg(&hb[(r0 + i) * 128 + m]);
      } else {
#pragma unroll
        for (int i = 0; i < NR; ++i) x[i] = 0.0f;
      }
    };
    const int hxo = lstm ? NR / 2 : NR;  // gst slot of hx (after the cell state)
    int hx_ep = -1;  // I_0 (split0): prediction epoch whose hh0 (from R_0, global) is in hx
    // R_0's hh0 MMA is read lazily: at the group's next use or when the next
    // round needs the accumulator (its group's registers / global state)
    int pend_r = -1, pend_g = 0;
    auto flush = [&]() {
      if (!r0m || pend_r < 0) return;
      float v[NR];
      read_acc(pend_r, v);
      if (pend_g == g) {
#pragma unroll
        for (int i = 0; i < NR; ++i) hx[i] = v[i];
      }
      if (P.ngrp > 1 || P.step_mode != STEP_NONE) {  // the group's state in global memory
        float* gs = P.gst + (((size_t)pend_g * P.G + blockIdx.x) * NSV + hxo) * NEPI + et;
#pragma unroll
        for (int i = 0; i < NR; ++i) gs[(size_t)i * NEPI] = v[i];
      }
      pend_r = -1;
    };
    run(
        [&](long long) {
          float v[NR], x[NR];
          if (c0) {
            flush();  // (normally done at the visit's start)
            if (!r0m && hx_ep != p) {  // I_0: hh0(p) from R_0 (P0: zeros)
              load_hh(p, hx);
              hx_ep = p;
            }
            // gates0 = (table0[label] + hh0) + b   (App. B order)
            if (p == 0) {  // P0: label blank for every row
#pragma unroll
              for (int i = 0; i < NR; ++i)
                ih[i] = r0 + i < B ? __ldg(&P.table0[(size_t)blank * P.GH + min(unit, P.Hp - 1) * P.Gg + gate]) : 0.0f;
            }
#pragma unroll
            for (int i = 0; i < NR; ++i) x[i] = (flag[r0 + i] & 2) ? ih[i] : 0.0f;
#pragma unroll
            for (int i = 0; i < NR; ++i) v[i] = (x[i] + hx[i]) + bias_m;
            mark(19);
          } else {
            post(p);
            load_hh(p, x);  // recurrent half from R_l, ready long before the input half
            read_acc(round - 1, v);
            mark(7);
            if (layer == 1) log_ld(48);
            if (PPROF(P) && layer == 1) log_chunks(92, clock64());
#pragma unroll
            for (int i = 0; i < NR; ++i) v[i] = (v[i] + x[i]) + bias_m;
          }
          if (lstm) cell_lstm(v, layer, p, c4, h4);
          else cell_tanh(v, layer, p, hr);
          mark_pub();
          gmark(c0 ? 44 : 46);
          mark(c0 ? 5 : 11);
          if (r0m) {
            // hh0 of the next prediction (h0(p) @ W_hh0): the MMA runs while the
            // rest of the step goes down the chain (and this CTA moves on)
            if (!wloaded) load_weights();
            post(p);
            pend_r = round - 1;
            pend_g = g;
          }
        },
        [&](long long) {
          if (r0m) flush();
        },
        [&](int mode) {
          if (mode == LD_INIT) {
#pragma unroll
            for (int j = 0; j < NR / 4; ++j) c4[j] = h4[j] = 0.0f;
#pragma unroll
            for (int j = 0; j < NR; ++j) hr[j] = hx[j] = 0.0f;
          } else if (mode == LD_MULTI) {
            if (lstm) {
#pragma unroll
              for (int j = 0; j < NR / 4; ++j) {
                c4[j] = *gstate(j);
                h4[j] = *gstate(NR / 4 + j);
              }
            } else {
#pragma unroll
              for (int j = 0; j < NR; ++j) hr[j] = *gstate(j);
            }
            if (r0m) {
#pragma unroll
              for (int j = 0; j < NR; ++j) hx[j] = *gstate(hxo + j);
            }
            hx_ep = -1;
          }
          if (mode == LD_INIT) hx_ep = -1;
          // merged R_0: the look-ahead hh0 MMA finished long ago; read it before
          // the decision so the layer-0 cell does not wait on the accumulator.
          // I_0: the next prediction's hh0 is ready long before the decision.
          if (r0m && mode != LD_INIT) flush();
          if (c0 && !r0m && mode != LD_INIT && hx_ep != p + 1) {
            load_hh(p + 1, hx);
            hx_ep = p + 1;
          }
        },
        [&]() {
          if (lstm) {
#pragma unroll
            for (int j = 0; j < NR / 4; ++j) {
              *gstate(j) = c4[j];
              *gstate(NR / 4 + j) = h4[j];
            }
          } else {
#pragma unroll
            for (int j = 0; j < NR; ++j) *gstate(j) = hr[j];
          }
          if (r0m && pend_r < 0) {  // (a pending hh0 is stored by its flush)
#pragma unroll
            for (int j = 0; j < NR; ++j) *gstate(hxo + j) = hx[j];
          }
        },
        nop);
    flush();  // merged R_0: the last look-ahead round
  }
  post(-1);
  if (P.ninst > 1 && (int)blockIdx.x == P.ic0[inst] && et == 0) {  // instance totals (Ctrl zeroed at launch)
    Ctrl* c = P.ctrl;
    atomicAdd(reinterpret_cast<unsigned long long*>(&c->joint_evals), (unsigned long long)joint_evals);
    atomicAdd(reinterpret_cast<unsigned long long*>(&c->pred_steps), (unsigned long long)pred_steps);
    atomicAdd(reinterpret_cast<unsigned long long*>(&c->outer_iters), (unsigned long long)outer_iters);
    atomicAdd(reinterpret_cast<unsigned long long*>(&c->iters), (unsigned long long)joint_evals);
    atomicMax(&c->err, err);
  } else if (P.ninst <= 1 && blockIdx.x == 0 && et == 0) {
    Ctrl* c = P.ctrl;
    c->joint_evals = joint_evals;
    c->pred_steps = pred_steps;
    c->outer_iters = outer_iters;
    c->iters = joint_evals;
    c->err = err;
  }
}

// ------------------------------------------------------------------ MMA round
// One load + MMA round of the MMA warp over chunks [0, KC): the first NLO
// chunks have W_lo in TMEM (TS x TS), the rest in smem (TS x SS); one elect
// per chunk issues its 8 MMAs and the stage commit.
template <int NLO, bool TR>
__device__ __forceinline__ void mma_round(const TParams& P, const Smem& sm, uint32_t& fb, int KC, uint32_t tmem,
                                          uint32_t whi0, uint32_t ring0, bool ctr, bool tr, int e) {
  constexpr uint32_t ID64 = idesc_f16(128, 64), ID32 = idesc_f16(128, 32);
  const uint32_t d1 = tmem, d2 = ACC64 ? tmem : tmem + 64;
  const uint32_t f2 = ACC64 ? 0u : 1u;  // (ACC64: the W_lo product always accumulates)
#pragma unroll  // (a rolled loop measured 0.45 us/step slower)
  for (int kc = 0; kc < MAXKC; ++kc) {
    if (kc < KC) {
      const int st = kc % NSTAGE;
      mbar_wait(&sm.full[st], (fb >> st) & 1u);
      fb ^= 1u << st;
      if (ctr) sm.dbg[16 + kc] = clock64();
      if (tr && (kc == 0 || kc == KC - 1)) PPROF(P)[(size_t)(kc ? 28 : 27) * PROF_WIN + (e - PROF_S0)] = gtimer();
      tc_fence_after();
      const uint64_t bd = sdesc_sw128(ring0 + st * CHUNK);
      if (kc < NLO)
        mma_chunk_tt2(d1, d2, tmem + WLO_COL + kc * 32, tmem + WLO_COL + (KC + kc) * 32, bd, kc == 0, ID64, ID32,
                      &sm.empty[st], f2 & (kc == 0));
      else
        mma_chunk_ts2(d1, d2, tmem + WLO_COL + kc * 32, sdesc_sw128(whi0 + kc * 16384), bd, kc == 0, ID64, ID32,
                      &sm.empty[st], f2 & (kc == 0));
    }
  }
}

// ------------------------------------------------------------------ kernel
#ifndef LB_THREADS
#define LB_THREADS NTH  // register budget = 65536 / LB_THREADS (A/B knob)
#endif
template <bool TR, int SPEC>
__global__ void __launch_bounds__(LB_THREADS, 1) ptc_kernel(const __grid_constant__ TParams P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  if (P.pdl) pdl_trigger();  // the next step launch may start its prologue on the free SMs
  unsigned long long t_entry = 0;
  if (STAMPS && threadIdx.x == 64) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_entry));
  const int4 rl = P.roles[blockIdx.x];
  const int role = rl.x, layer = rl.y & 0xff, inst = rl.y >> 8, tile = rl.z;
  const float wsc = __int_as_float(rl.w);
  const int in_buf = (role == ROLE_J || role == ROLE_E) ? TRUNK : role == ROLE_P ? P.L - 1 : role == ROLE_R ? layer
                                                                                                      : max(layer - 1, 0);
  const int KC = (role == ROLE_E || (role == ROLE_I && layer == 0)) ? 0 : P.act_kc[in_buf];  // no weights: E, I_0
  Smem sm = carve(smem_raw, KC);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const CfgFlags<SPEC> cf(P);
  const bool lstm = cf.lstm, fs = cf.fs, tdt = cf.tdt;

  if (tid == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.accf[i], 1);
      mbar_init(&sm.acce[i], NEPI / 32);
    }
    mbar_init(sm.cmd, 1);
    mbar_init(sm.wbar, 1);
    mbar_init(sm.wready, NEPI / 32);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sm.tslot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *sm.tslot;
  const unsigned char* wimg = P.wimg + (size_t)blockIdx.x * P.wstride;

  // ---- resident weights: W_hi -> smem (bulk copies), W_lo -> TMEM ----
#ifndef XP_NOWLO
#define XP_NOWLO 0  // timing experiments only (wrong results): skip the smem weight copy
#endif
#ifndef WCOPY_ALL
#define WCOPY_ALL 0  // A/B: copy the TMEM-resident chunks' W_lo into smem too (round-2 layout)
#endif
#ifndef XP_NOWHI
#define XP_NOWHI 0  // timing experiments only: skip the TMEM weight load
#endif
  if (tid == 0) {
    // the first nlo_chunks(KC) chunks' W_lo is TMEM-resident (loaded by the
    // epilogue): only the rest of the image goes to smem
    const uint32_t o0 = KC && !WCOPY_ALL ? (uint32_t)nlo_chunks(KC) * 16384 : 0u;
    const uint32_t bytes = XP_NOWLO ? o0 : (uint32_t)KC * 16384;
    mbar_arrive_expect_tx(sm.wbar, bytes - o0);
    for (uint32_t o = o0; o < bytes; o += 32768)
      bulk_g2s(sm.whi + o, wimg + o, bytes - o < 32768 ? bytes - o : 32768, sm.wbar);
  }

  if (warp == 0) {
    // ================= producer (converged warp): stream input chunks into the ring =================
    // Stage of chunk kc is kc % NSTAGE every round: a round is posted only after
    // the epilogue read the previous round's accumulator, so every earlier MMA
    // (and its smem read) has completed and the first NSTAGE chunks' empty-
    // barrier waits return at once (they are still made, so every phase of
    // every barrier is waited on: compute-sanitizer synccheck clean).
    // eb bit s = uses of stage s so far (mod 2).
    const unsigned* mycnt0 = P.cnt + (size_t)(cidx_act(in_buf, 0) + (lane < KC ? lane : 0)) * CSTRIDE;
    const unsigned my_np = lane < KC ? (unsigned)P.nprod[in_buf][lane] : 0u;
    const CUtensorMap* lmap = &P.ldmap[in_buf];
    const bool stamp_ip = PPROF(P) && (role == ROLE_I || role == ROLE_P) && (int)blockIdx.x == P.prof_first[role];
    const bool ctr = PPROF(P) && (role == ROLE_J || role == ROLE_I) && (int)blockIdx.x == P.prof_first[role] && lane == 0;
    const bool trj = PPROF(P) && role == ROLE_J && (int)blockIdx.x == P.prof_first[role] && lane == 0;
    unsigned long long* const prof = PPROF(P);
    const uint32_t ring0 = smem_u32(sm.ring);
    uint32_t eb = 0, used = 0;
    for (int r = 0;; ++r) {
      mbar_wait(sm.cmd, r & 1);
      const int e = ((volatile int*)sm.misc)[r & 1];
      if (e < 0) break;
      const int grp = ((volatile int*)sm.misc)[6 + (r & 1)];  // the round's row group
      const unsigned* mycnt = mycnt0 + (size_t)grp * NCOUNTERS * CSTRIDE;
      const bool tr = trj && e >= PROF_S0 && e < PROF_S0 + PROF_WIN;
      const unsigned target = my_np * (unsigned)(e + 1);
      int next = 0, npoll = 0;
      while (next < KC) {
        // one counter per lane, all in flight in one instruction
        const bool need = lane >= next && lane < KC;
        unsigned v = 0u;
        if (need) v = ld_poll_cnt(mycnt);
        const unsigned ok = __ballot_sync(0xffffffffu, lane < next || (need && v >= target));
        const int ready = __ffs(~ok) - 1;  // chunks [0, ready) are published
        if (ctr) ++npoll;
        if (ready == next) continue;
        if (ctr && next == 0) sm.dbg[10] = npoll;
        // relaxed counter reads + a fence / acquire re-read (warp-synchronised:
        // any lane may issue the loads below): the acquire pattern
        if (MM_CONS == 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (MM_CONS == 4) asm volatile("fence.acquire.gpu;" ::: "memory");
        if (MM_CONS == 3) {
          if (lane >= next && lane < ready) acquire_after(mycnt);
          __syncwarp();
        }
        fence_proxy_global();
#pragma unroll
        for (int kc = 0; kc < MAXKC; ++kc) {
          if (kc >= next && kc < ready) {
            const int st = kc % NSTAGE;
            // every phase of a stage's empty barrier is waited on once (the
            // first NSTAGE chunks of a round find theirs complete: the round was
            // posted after the epilogue read the previous round's accumulator)
            if ((used >> st) & 1u) mbar_wait(&sm.empty[st], ((eb >> st) & 1u) ^ 1u);
            used |= 1u << st;
            eb ^= 1u << st;
            if (tr && (kc == 0 || kc == KC - 1)) prof[(size_t)(kc ? 13 : 12) * PROF_WIN + (e - PROF_S0)] = gtimer();
            if ((kc == 0 || kc == KC - 1) && stamp_ip && lane == 0)
              reinterpret_cast<volatile unsigned long long*>(sm.misc + 8)[kc ? 1 : 0] = gtimer();
            if (ctr) sm.dbg[kc] = clock64();
            if (elect_one()) {
              mbar_arrive_expect_tx(&sm.full[st], CHUNK);
              tma_ld2_u(ring0 + st * CHUNK, lmap, 64 * kc, 64 * (2 * grp + (e & 1)), &sm.full[st]);
            }
            __syncwarp();
          }
        }
        next = ready;
      }
      if (ctr) sm.dbg[11] = npoll;
    }
    // a step launch may end without an MMA round: the smem weight copy must
    // still land before the CTA exits (no async write may outlive it)
    mbar_wait(sm.wbar, 0);
  } else if (warp == 1) {
    // ================= MMA issuer (converged warp) =================
    const uint32_t whi0 = smem_u32(sm.whi), ring0 = smem_u32(sm.ring);
    const bool ctr = PPROF(P) && (role == ROLE_J || role == ROLE_I) && (int)blockIdx.x == P.prof_first[role] && lane == 0;
    const bool trj = PPROF(P) && role == ROLE_J && (int)blockIdx.x == P.prof_first[role] && lane == 0;
    const bool stamp_ip = PPROF(P) && (role == ROLE_I || role == ROLE_P) && (int)blockIdx.x == P.prof_first[role] && lane == 0;
    uint32_t fb = 0;  // bit s = fills of stage s consumed so far (mod 2)
    const int nlo = nlo_chunks(KC);
    for (int r = 0;; ++r) {
      mbar_wait(sm.cmd, r & 1);
      const int e = ((volatile int*)sm.misc)[r & 1];
      if (e < 0) break;
      if (r == 0) {  // the weights, before the first MMA
        mbar_wait(sm.wbar, 0);    // W_lo smem image
        mbar_wait(sm.wready, 0);  // TMEM weights (the epilogue's first post)
        tc_fence_after();
      }
      const int set = 0;
      if (r >= 1) mbar_wait(&sm.acce[0], (uint32_t)((r - 1) & 1));  // the epilogue read the last round
      tc_fence_after();
      const bool tr = trj && e >= PROF_S0 && e < PROF_S0 + PROF_WIN;
      switch (nlo) {  // once per round: no per-chunk branch between the two MMA forms
        case 0: mma_round<0, TR>(P, sm, fb, KC, tmem, whi0, ring0, ctr, tr, e); break;
        case 1: mma_round<1, TR>(P, sm, fb, KC, tmem, whi0, ring0, ctr, tr, e); break;
        case 2: mma_round<2, TR>(P, sm, fb, KC, tmem, whi0, ring0, ctr, tr, e); break;
        case 3: mma_round<3, TR>(P, sm, fb, KC, tmem, whi0, ring0, ctr, tr, e); break;
        case 4: mma_round<4, TR>(P, sm, fb, KC, tmem, whi0, ring0, ctr, tr, e); break;
        case 5: mma_round<5, TR>(P, sm, fb, KC, tmem, whi0, ring0, ctr, tr, e); break;
        case 6: mma_round<6, TR>(P, sm, fb, KC, tmem, whi0, ring0, ctr, tr, e); break;
        default: mma_round<MAXNLO, TR>(P, sm, fb, KC, tmem, whi0, ring0, ctr, tr, e); break;
      }
      mma_commit(&sm.accf[set]);
      if (ctr) sm.dbg[31] = clock64();
      if (tr) PPROF(P)[(size_t)29 * PROF_WIN + (e - PROF_S0)] = gtimer();
      if (stamp_ip) reinterpret_cast<volatile unsigned long long*>(sm.misc + 8)[2] = gtimer();
    }
  } else {
    // ================= epilogue + replicated control (128 threads) =================
    Epi<TR, SPEC> e(P, sm, tmem, tid - 64, warp & 3, role, layer, tile, inst, wsc);
    e.t_entry = t_entry;
    e.run_role();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace ptc
}  // namespace rnntg
