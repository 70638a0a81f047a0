// rnntg.cu — host side of the C ABI (include/rnntg.h): weight repacking,
// static device workspaces, CUDA-graph construction with nested conditional
// WHILE nodes, launch / read, and the kernel-level step entry points.
//
// Reference mapping (decoders.hpp:56-130):
//   rnntg_decoder_create   build_decode_graph   (decoders.cpp:589-627)
//   rnntg_bind             bind_decode_inputs   (decoders.cpp:202-207, 124-142)
//   rnntg_launch           Engine::replay       (engine.cpp:296-307)
//   rnntg_read             read_emissions       (decoders.cpp:97-122)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rnntg.h"
#include "common.cuh"
#include "kernels.cuh"
#include "encproj_tc.cuh"
#include "persistent_k5.cuh"
#include "persistent_tc.cuh"

using namespace rnntg;

namespace rnntg {
// ptc_kernels.cu (its own translation unit: ptxas -O1, see the Makefile)
const void* tc_kernel_for(int algo, int cell, bool traced);
}  // namespace rnntg

namespace {

thread_local std::string g_err;

rnntg_status fail(rnntg_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CK(expr)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(RNNTG_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));    \
  } while (0)

int round_up(int x, int m) { return (x + m - 1) / m * m; }

bool env_flag(const char* name, bool dflt) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  return !(v[0] == '0' || v[0] == 'n' || v[0] == 'N' || v[0] == 'f' || v[0] == 'F');
}

struct DevBuf {
  std::vector<void*> ptrs;
  template <typename T>
  cudaError_t alloc(T** p, size_t n) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T));
    if (e != cudaSuccess) return e;
    ptrs.push_back(q);
    *p = static_cast<T*>(q);
    return cudaMemset(q, 0, std::max<size_t>(n, 1) * sizeof(T));
  }
  void release() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
  }
};

}  // namespace

struct rnntg_model {
  int device = 0;
  rnntg_dims dims{};
  DevModel dm{};
  DevBuf mem;
  std::vector<std::vector<float>> host_w;  // reference-order weights (persistent packing)
  bool tc_ok = false;   // tcgen05 encoder projection usable on this device
};

struct rnntg_decoder {
  rnntg_model* m = nullptr;
  int algo = 0, exec = 0, B = 0, T = 0, ms = 0;
  DevState st{};
  DevBuf mem;
  cudaStream_t stream = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  // persistent executors: encoder projection + counter resets + the
  // cooperative kernel captured once, replayed by one cudaGraphLaunch (the
  // host otherwise leaves the GPU idle between the projection and the
  // persistent kernel for the duration of the cooperative-launch call)
  cudaGraphExec_t lexec = nullptr;
  bool ltried = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool bound = false, launched = false;
  float* x_dev = nullptr;  // [B*T][Fp] pitched, zero-padded features
  EncPlan enc;             // K1 tensor maps over x_dev -> st.fp
  int* len_dev = nullptr;
  int* len_bad = nullptr;  // set on the device when bound device lengths lie outside [0, T]
  // kernel-node argument storage (copied into the nodes at creation)
  DevModel arg_m{};
  DevState arg_s{};
  int arg_l[MAXL]{};
  // persistent executor
  pk::PParams pp{};
  size_t psmem = 0;
  // tensor-core persistent executor
  ptc::TParams tp{};
  // graph / host-loop executors on the tensor-core step kernel: the init and
  // one-step launch parameters (tp with step_mode STEP_INIT / STEP_ONE)
  bool tc_steps = false;
  ptc::TParams tp_step[2]{};
  size_t tsmem = 0;
  unsigned* tcnt = nullptr;
  size_t tcnt_bytes = 0, tpw_bytes = 0;
  // sync-requiring host-loop baseline: pinned mirror of the control block
  Ctrl* hctrl = nullptr;
  // host-side work of the last decode (TimingReport.num_syncs / launches)
  int64_t n_syncs = 0, n_launches = 0, n_graph_launches = 0;
  // tensor executor above its per-kernel batch: balanced sub-batches of
  // <= ptc::MAXB * ptc::MAXG rows, each its own tensor-core decoder, run back to back on
  // this decoder's stream (every K6 kernel takes most of the GPU's SMs)
  std::vector<rnntg_decoder*> subs;
  std::vector<int> sub_b0;
  bool owns_stream = true;
};

namespace {

// ---------------------------------------------------------------- model
rnntg_status validate_dims(const rnntg_dims* d) {
  if (!d) return fail(RNNTG_E_VALUE, "dims is null");
  if (d->vocab < 1 || d->embed < 1 || d->hidden < 1 || d->joint < 1 || d->feature < 1)
    return fail(RNNTG_E_VALUE, "all transducer dimensions must be >= 1");
  if (d->cell != RNNTG_CELL_TANH && d->cell != RNNTG_CELL_LSTM)
    return fail(RNNTG_E_VALUE, "unknown cell");
  if (d->layers < 1 || d->layers > RNNTG_MAX_LAYERS)
    return fail(RNNTG_E_VALUE, "layers must lie in [1, 4]");
  if (d->cell == RNNTG_CELL_TANH && d->layers != 1)
    return fail(RNNTG_E_VALUE, "the tanh prediction network has exactly one layer");
  if (d->num_durations < 0 || d->num_durations > RNNTG_MAX_DURATIONS)
    return fail(RNNTG_E_VALUE, "too many duration classes");
  if (d->num_durations > 0) {  // model.cpp:69-78
    if (d->durations[0] != 0 && d->durations[0] != 1)
      return fail(RNNTG_E_VALUE, "first duration must be 0 or 1");
    for (int i = 1; i < d->num_durations; ++i)
      if (d->durations[i] <= d->durations[i - 1])
        return fail(RNNTG_E_VALUE, "durations must be strictly ascending");
  }
  return RNNTG_OK;
}

int num_weights(const rnntg_dims* d) { return 1 + 3 * d->layers + 3 + (d->num_durations > 0); }

// [K][N] row-major -> [N/CT][K][CT]: each step-GEMV tile's weights (and every
// warp's k-slice of them) become one contiguous block for bulk copies.
std::vector<float> tile16(const std::vector<float>& W, int K, int N) {
  std::vector<float> T(W.size());
  for (int t = 0; t < N / CT; ++t)
    for (int k = 0; k < K; ++k)
      for (int c = 0; c < CT; ++c)
        T[((size_t)t * K + k) * CT + c] = W[(size_t)k * N + t * CT + c];
  return T;
}

template <typename T>
cudaError_t upload(DevBuf& mem, T** dst, const std::vector<T>& src) {
  cudaError_t e = mem.alloc(dst, src.size());
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice);
}

// ---------------------------------------------------------------- state
rnntg_status alloc_state(rnntg_model* m, DevBuf& mem, DevState& s, int algo, int B, int T,
                         int ms, bool debug) {
  const DevModel& M = m->dm;
  s = DevState{};
  s.B = B;
  s.Bp = round_up(B, RB);
  s.nrb = s.Bp / RB;
  s.T = T;
  s.ms = ms;
  s.cap = std::max(1, T * ms);
  s.algo = algo;
  s.max_iters = 1000000;  // engine.hpp:249 default while-iteration cap
  const size_t Bp = s.Bp;
  CK(mem.alloc(&s.fp, (size_t)B * T * M.Jp));
  for (int l = 0; l < M.L; ++l)
    for (int p = 0; p < 2; ++p) {
      CK(mem.alloc(&s.h[l][p], Bp * M.Hp));
      if (M.cell == RNNTG_CELL_LSTM) CK(mem.alloc(&s.c[l][p], Bp * M.Hp));
    }
  CK(mem.alloc(&s.gp, Bp * M.Jp));
  int* ints = nullptr;
  CK(mem.alloc(&ints, Bp * 8));
  s.last_label = ints;
  s.accept = ints + Bp;
  s.done = ints + 2 * Bp;
  s.need = ints + 3 * Bp;
  s.active = ints + 4 * Bp;
  s.t_row = ints + 5 * Bp;
  s.u_row = ints + 6 * Bp;
  s.counts = ints + 7 * Bp;
  CK(mem.alloc(&s.tokens, (size_t)B * s.cap));
  CK(mem.alloc(&s.frames, (size_t)B * s.cap));
  CK(mem.alloc(&s.scores, (size_t)B * s.cap));
  CK(mem.alloc(&s.durs, (size_t)B * s.cap));
  CK(mem.alloc(&s.part, Bp * M.NCHT));
  CK(mem.alloc(&s.ctrl, 1));
  if (debug) {
    CK(mem.alloc(&s.dbg_logits, Bp * M.NOUT));
    CK(mem.alloc(&s.dbg_lse, 2 * Bp));
  }
  return RNNTG_OK;
}

size_t joint_smem(const DevModel& M) { return step_smem_bytes(M.Jp); }
size_t layer_smem(const DevModel& M, int l) { return step_smem_bytes(l == 0 ? M.Hp : 2 * M.Hp); }
size_t pp_smem(const DevModel& M) { return step_smem_bytes(M.Hp); }

cudaError_t set_smem_attrs(const DevModel& M) {
  // The attribute belongs to the kernel, not to a model: set the device
  // maximum so a smaller model created later cannot lower it below what an
  // earlier, larger model's launches need.
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) !=
      cudaSuccess)
    return e;
  const int need = (int)std::max({joint_smem(M), layer_smem(M, 1), layer_smem(M, 0), pp_smem(M)});
  if (need > optin) return cudaErrorInvalidValue;
  const int big = optin;
  if ((e = cudaFuncSetAttribute(pred_layer_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                big)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(pred_layer_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                big)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(pred_proj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                big)) != cudaSuccess)
    return e;
  return cudaFuncSetAttribute(joint_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
}

// ---------------------------------------------------------------- graph
struct Builder {
  cudaGraph_t g;
  cudaGraphNode_t last = nullptr;
  bool last_kernel = false;
  bool pdl = true;

  cudaError_t kernel(const void* fn, dim3 grid, dim3 block, size_t smem, void** args) {
    cudaGraphNodeParams p{};
    p.type = cudaGraphNodeTypeKernel;
    p.kernel.func = const_cast<void*>(fn);
    p.kernel.gridDim = grid;
    p.kernel.blockDim = block;
    p.kernel.sharedMemBytes = (unsigned)smem;
    p.kernel.kernelParams = args;
    cudaGraphEdgeData e{};
    if (pdl && last_kernel) {
      e.from_port = cudaGraphKernelNodePortProgrammatic;
      e.type = cudaGraphDependencyTypeProgrammatic;
    }
    cudaGraphNode_t n;
    cudaError_t err = cudaGraphAddNode_v2(&n, g, last ? &last : nullptr, last ? &e : nullptr,
                                          last ? 1 : 0, &p);
    if (err != cudaSuccess) return err;
    last = n;
    last_kernel = true;
    return cudaSuccess;
  }

  cudaError_t while_node(cudaGraphConditionalHandle h, cudaGraph_t* body) {
    cudaGraphNodeParams p{};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t n;
    cudaError_t err = cudaGraphAddNode(&n, g, last ? &last : nullptr, last ? 1 : 0, &p);
    if (err != cudaSuccess) return err;
    *body = p.conditional.phGraph_out[0];
    last = n;
    last_kernel = false;
    return cudaSuccess;
  }
};

void* kargs2(DevModel* m, DevState* s, void** out) {
  out[0] = m;
  out[1] = s;
  return out;
}

// Adds the prediction step: L layer kernels + pred_proj.
cudaError_t add_pred_step(Builder& b, rnntg_decoder* d) {
  const DevModel& M = d->m->dm;
  const int nrb = d->st.nrb;
  cudaError_t e;
  if (M.cell == RNNTG_CELL_SCRIPTED) {
    void* args[2] = {&d->arg_m, &d->arg_s};
    return b.kernel((const void*)scripted_pred_kernel, dim3(1), dim3(NT), 0, args);
  }
  for (int l = 0; l < M.L; ++l) {
    void* args[3] = {&d->arg_m, &d->arg_s, &d->arg_l[l]};
    const void* fn = M.cell == RNNTG_CELL_LSTM ? (const void*)pred_layer_kernel<1>
                                               : (const void*)pred_layer_kernel<0>;
    if ((e = b.kernel(fn, dim3(M.GH / CT, nrb), dim3(NT), layer_smem(M, l), args)) != cudaSuccess)
      return e;
  }
  void* args[2] = {&d->arg_m, &d->arg_s};
  return b.kernel((const void*)pred_proj_kernel, dim3(M.Jp / CT, nrb), dim3(NT), pp_smem(M), args);
}

cudaError_t add_joint(Builder& b, rnntg_decoder* d) {
  const DevModel& M = d->m->dm;
  void* args[2] = {&d->arg_m, &d->arg_s};
  return b.kernel((const void*)joint_kernel, dim3(M.NCHT, d->st.nrb), dim3(NT), joint_smem(M),
                  args);
}

cudaError_t add_encproj(Builder& b, rnntg_decoder* d);

// Persistent executor setup: per-CTA weight packing (resident in shared
// memory for the whole decode), chunk-major activation buffers, checks that
// the model fits (LSTM <= 2 layers or tanh, batch <= 256, smem budget).
rnntg_status setup_persistent(rnntg_decoder* d) {
  rnntg_model* m = d->m;
  const DevModel& M = m->dm;
  const rnntg_dims& dd = m->dims;
  const bool lstm = M.cell == RNNTG_CELL_LSTM;
  if (M.L > 2) return fail(RNNTG_E_VALUE, "persistent executor supports at most 2 layers");
  if (d->B > pk::MAXB) return fail(RNNTG_E_VALUE, "persistent executor supports batch <= 256");
  const int umax = lstm ? pk::UMAX_LSTM : pk::UMAX_TANH;
  const int H = M.H, J = M.J, V1 = M.V1, D = M.D, NJ = V1 + D, Hp = M.Hp, Jp = M.Jp;
  const int Gc = lstm ? 4 : 1;
  int G = std::max({(H + umax - 1) / umax, (J + pk::C2 - 1) / pk::C2, (NJ + pk::C2 - 1) / pk::C2, 1});
  int nsm = 0, optin = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device));
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, m->device));
  if (G > nsm) return fail(RNNTG_E_VALUE, "model too wide for the persistent executor");
  const int wfloats = Hp * pk::C1 + (M.L == 2 ? 2 * Hp * pk::C1 : 0) + Hp * pk::C2 + Jp * pk::C2;
  // Per-warp activation slot (ns*8 features) and the CTA-private own-state:
  // prefer own-state in shared memory (saves L2 round trips in every
  // epilogue), then the largest slot that still fits.
  const size_t ownf = pk::own_floats(d->B, umax);
  int ns = 0, own = 0;
  for (int o = 1; o >= 0 && !ns; --o)
    for (int cand = pk::MAX_NS; cand >= 3 && !ns; --cand)
      if (pk::smem_bytes(wfloats, cand, d->B, o ? ownf : 0) <= (size_t)optin) {
        ns = cand;
        own = o;
      }
  for (int cand = pk::MAX_NS; cand >= 2 && !ns; --cand)
    if (pk::smem_bytes(wfloats, cand, d->B) <= (size_t)optin) ns = cand;
  if (const char* e = std::getenv("RNNTG_NS")) {
    const int want = std::atoi(e);
    if (want >= 2 && want <= pk::MAX_NS &&
        pk::smem_bytes(wfloats, want, d->B, own ? ownf : 0) <= (size_t)optin)
      ns = want;
  }
  if (env_flag("RNNTG_OWN_GLOBAL", false)) own = 0;
  if (!ns) return fail(RNNTG_E_VALUE, "persistent executor: weights exceed shared memory");
  d->psmem = pk::smem_bytes(wfloats, ns, d->B, own ? ownf : 0);
  // per-kernel attribute shared by all decoders: set the device maximum
  CK(cudaFuncSetAttribute(pk::persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          optin));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pk::persistent_kernel, pk::NTH,
                                                   d->psmem));
  if (per_sm < 1 || G > per_sm * nsm)
    return fail(RNNTG_E_VALUE, "persistent executor cannot be co-resident");
  // ---- pack weights per CTA ----
  const auto& w = m->host_w;
  const int L = M.L, bse = 1 + 3 * L;
  const int off_hh0 = 0, off_w1 = Hp * pk::C1, off_pp = off_w1 + (L == 2 ? 2 * Hp * pk::C1 : 0),
            off_j = off_pp + Hp * pk::C2;
  std::vector<float> pack((size_t)G * wfloats, 0.0f), bias((size_t)G * 2 * pk::C1, 0.0f);
  for (int c = 0; c < G; ++c) {
    float* P = pack.data() + (size_t)c * wfloats;
    const int u0 = pk::own_lo(H, c, G), u1 = pk::own_lo(H, c + 1, G);
    for (int lu = 0; lu < u1 - u0; ++lu)
      for (int g = 0; g < Gc; ++g) {
        const int col = lu * Gc + g, rc = g * H + u0 + lu;
        for (int k = 0; k < H; ++k) {
          P[off_hh0 + k * pk::C1 + col] = w[2][(size_t)k * Gc * H + rc];
          if (L == 2) {
            P[off_w1 + k * pk::C1 + col] = w[4][(size_t)k * Gc * H + rc];
            P[off_w1 + (Hp + k) * pk::C1 + col] = w[5][(size_t)k * Gc * H + rc];
          }
        }
        bias[(size_t)c * 2 * pk::C1 + col] = w[3][rc];
        if (L == 2) bias[(size_t)c * 2 * pk::C1 + pk::C1 + col] = w[6][rc];
      }
    const int p0 = pk::own_lo(J, c, G), p1 = pk::own_lo(J, c + 1, G);
    for (int k = 0; k < H; ++k)
      for (int lj = 0; lj < p1 - p0; ++lj) P[off_pp + k * pk::C2 + lj] = w[bse + 1][(size_t)k * J + p0 + lj];
    const int n0 = pk::own_lo(NJ, c, G), n1 = pk::own_lo(NJ, c + 1, G);
    for (int k = 0; k < J; ++k)
      for (int ln = 0; ln < n1 - n0; ++ln) {
        const int n = n0 + ln;
        P[off_j + k * pk::C2 + ln] =
            n < V1 ? w[bse + 2][(size_t)k * V1 + n] : w[bse + 3][(size_t)k * D + (n - V1)];
      }
  }
  pk::PParams& pp = d->pp;
  pp = pk::PParams{};
  pp.G = G;
  pp.B = d->B;
  pp.nrb = d->st.nrb;
  pp.T = d->T;
  pp.ms = d->ms;
  pp.cap = d->st.cap;
  pp.algo = d->algo;
  pp.L = L;
  pp.cell = M.cell;
  pp.H = H;
  pp.Hp = Hp;
  pp.J = J;
  pp.Jp = Jp;
  pp.V1 = V1;
  pp.D = D;
  pp.NJ = NJ;
  pp.ns = ns;
  pp.own_smem = own;
  pp.max_iters = d->st.max_iters;
  for (int i = 0; i < D; ++i) pp.durations[i] = dd.durations[i];
  pp.wfloats = wfloats;
  pp.off_hh0 = off_hh0;
  pp.off_w1 = off_w1;
  pp.off_pp = off_pp;
  pp.off_j = off_j;
  pp.GH = M.GH;
  pp.Gg = M.G;
  pp.table0 = M.table0;
  float* dp = nullptr;
  CK(upload(d->mem, &dp, pack));
  pp.wpack = dp;
  CK(upload(d->mem, &dp, bias));
  pp.bias = dp;
  const size_t Bp = d->st.Bp;
  CK(d->mem.alloc(&pp.h0, Bp * Hp));
  CK(d->mem.alloc(&pp.h1[0], Bp * Hp));
  CK(d->mem.alloc(&pp.h1[1], Bp * Hp));
  CK(d->mem.alloc(&pp.trunk, Bp * Jp));
  CK(d->mem.alloc(&pp.hh0own, (size_t)G * d->B * pk::C1));
  CK(d->mem.alloc(&pp.cown, (size_t)G * 2 * d->B * pk::UMAX_TANH));
  CK(d->mem.alloc(&pp.gpown, (size_t)G * d->B * pk::C2));
  CK(d->mem.alloc(&pp.partv, (size_t)G * d->B));
  CK(d->mem.alloc(&pp.partd, (size_t)G * d->B));
  CK(d->mem.alloc(&pp.amax, (size_t)2 * d->B));
  CK(d->mem.alloc(&pp.dmax, (size_t)2 * d->B));
  CK(d->mem.alloc(&pp.bar, 2));
  if (env_flag("RNNTG_PROF", false)) CK(d->mem.alloc(&pp.prof, 16));
  // CTAs owning duration-head columns (joint columns >= V1)
  pp.dc0 = G;
  pp.dc1 = G;
  for (int c = 0; c < G; ++c)
    if (pk::own_lo(NJ, c + 1, G) > V1) {
      pp.dc0 = c;
      break;
    }
  pp.fp = d->st.fp;
  pp.out_len = d->len_dev;
  pp.tokens = d->st.tokens;
  pp.frames = d->st.frames;
  pp.scores = d->st.scores;
  pp.durs = d->st.durs;
  pp.counts = d->st.counts;
  pp.ctrl = d->st.ctrl;
  (void)Gc;
  return RNNTG_OK;
}

// ---------------------------------------------------------------- K6
// fp16 bits (round to nearest even) of a float, host side.
uint16_t f2h_bits(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const int exp = (int)((x >> 23) & 0xff) - 127 + 15;
  uint32_t mant = x & 0x7fffffu;
  if (((x >> 23) & 0xff) == 0xff) return (uint16_t)(sign | 0x7c00u | (mant ? 0x200u : 0));
  if (exp >= 31) return (uint16_t)(sign | 0x7c00u);
  if (exp <= 0) {
    if (exp < -10) return (uint16_t)sign;
    mant |= 0x800000u;
    const int shift = 14 - exp;
    uint32_t h = mant >> shift;
    const uint32_t rem = mant & ((1u << shift) - 1), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (h & 1))) ++h;
    return (uint16_t)(sign | h);
  }
  uint32_t h = ((uint32_t)exp << 10) | (mant >> 13);
  const uint32_t rem = mant & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1))) ++h;
  return (uint16_t)(sign | h);
}
float h2f(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const int exp = (h >> 10) & 0x1f;
  uint32_t mant = h & 0x3ffu;
  uint32_t x;
  if (exp == 0) {
    if (!mant) x = sign;
    else {
      int e = -1;
      do { mant <<= 1; ++e; } while (!(mant & 0x400u));
      x = sign | ((uint32_t)(127 - 15 - e) << 23) | ((mant & 0x3ffu) << 13);
    }
  } else if (exp == 31) x = sign | 0x7f800000u | (mant << 13);
  else x = sign | ((uint32_t)(exp - 15 + 127) << 23) | (mant << 13);
  float f;
  std::memcpy(&f, &x, 4);
  return f;
}

// Tensor-core persistent executor: role assignment (one 128-row weight tile
// per CTA), fp16 hi/lo weight images, activation / counter buffers.
rnntg_status setup_tc(rnntg_decoder* d, bool allow_inst = true) {
  rnntg_model* m = d->m;
  const DevModel& M = m->dm;
  const rnntg_dims& dd = m->dims;
  const bool lstm = M.cell == RNNTG_CELL_LSTM;
  const int H = M.H, J = M.J, V1 = M.V1, D = M.D, Hp = M.Hp, Jp = M.Jp, L = M.L;
  if (d->B > ptc::MAXB * ptc::MAXG) return fail(RNNTG_E_VALUE, "tensor-core executor supports batch <= 256");
  const int ngrp = (d->B + ptc::MAXB - 1) / ptc::MAXB;  // balanced row groups of <= 32 rows
  if (Hp > ptc::MAXKP || Jp > ptc::MAXKP)
    return fail(RNNTG_E_VALUE, "tensor-core executor supports hidden/joint <= 640");
  const int NJ = (V1 + D + 127) / 128, NP = (J + 127) / 128;
  const int NG = lstm ? (H + 31) / 32 : (H + 127) / 128;
  if (NJ > ptc::MAXNJ) return fail(RNNTG_E_VALUE, "tensor-core executor: vocab + durations <= 2048");
  if (NG > 64) return fail(RNNTG_E_VALUE, "tensor-core executor: too many gate tiles");
  int nsm = 0, optin = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device));
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, m->device));
  // split0: the layer-0 cell on its own (weightless) I_0 CTAs and the
  // hypotheses on an emitter CTA (E) -- the shortest per-step chain; else the
  // cell merged into R_0 and the emitter into R_{L-1} tile 0 (fewer CTAs).
  // Two row groups or more and room for two merged CTA sets: two instances,
  // each decoding half of the groups on its own SMs.
  const int g_merged = NJ + NP + NG * (2 * L - 1);
  const int ninst = allow_inst && ngrp >= 2 && 2 * g_merged <= nsm && !env_flag("RNNTG_ONE_INST", false) ? 2 : 1;
  const int split0 = ninst > 1 || env_flag("RNNTG_MERGE0", false) ? 0 : 1;
  std::vector<int4> roles;
  int ic0[ptc::MAXI + 1] = {0, 0, 0};
  for (int i = 0; i < ninst; ++i) {
    ic0[i] = (int)roles.size();
    for (int t = 0; t < NJ; ++t) roles.push_back(make_int4(ptc::ROLE_J, i << 8, t, 0));
    for (int t = 0; t < NP; ++t) roles.push_back(make_int4(ptc::ROLE_P, i << 8, t, 0));
    for (int l = 0; l < L; ++l) {
      for (int t = 0; t < NG; ++t) roles.push_back(make_int4(ptc::ROLE_R, l | (i << 8), t, 0));
      if (l > 0 || split0)
        for (int t = 0; t < NG; ++t) roles.push_back(make_int4(ptc::ROLE_I, l | (i << 8), t, 0));
    }
    if (split0) roles.push_back(make_int4(ptc::ROLE_E, i << 8, 0, 0));
  }
  ic0[ninst] = (int)roles.size();
  const int G = (int)roles.size();
  if (G > nsm) return fail(RNNTG_E_VALUE, "tensor-core executor needs one SM per weight tile");
  const int KCmax = std::max(Hp, Jp) / 64;
  d->tsmem = ptc::smem_bytes(KCmax);
  if (d->tsmem > (size_t)optin) return fail(RNNTG_E_VALUE, "tensor-core executor: smem budget");
  CK(cudaFuncSetAttribute(tc_kernel_for(d->algo, M.cell, false), cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
  CK(cudaFuncSetAttribute(tc_kernel_for(d->algo, M.cell, true), cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tc_kernel_for(d->algo, M.cell, false), ptc::NTH,
                                                   d->tsmem));
  if (per_sm < 1) return fail(RNNTG_E_VALUE, "tensor-core executor cannot be resident");
  // ---- weight images: W_hi [KC][128 x 64] swizzled, then W_lo [K/2][128] packed pairs ----
  const auto& w = m->host_w;
  const int bse = 1 + 3 * L;
  // per CTA: [KCmax][16 KB] smem image, then TMEM column pairs (u32 = 2 fp16
  // along k) for 128 lanes: the KC chunks' TMEM-resident half, then W_lo of
  // the first nlo_chunks(KC) chunks
  const size_t wtoff = (size_t)KCmax * 16384;
  int tcols = 0;
  for (int kc : {Hp / 64, Jp / 64}) tcols = std::max(tcols, (kc + ptc::nlo_chunks(kc)) * 32);
  const size_t wstride = wtoff + (size_t)tcols * 128 * 4;
  std::vector<unsigned char> img((size_t)G * wstride, 0);
  std::vector<float> row(ptc::MAXKP);
  for (int c = 0; c < G; ++c) {
    const int role = roles[c].x, l = roles[c].y & 0xff, t = roles[c].z;
    if (role == ptc::ROLE_E || (role == ptc::ROLE_I && l == 0)) {  // no weights
      const float one = 1.0f;
      std::memcpy(&roles[c].w, &one, 4);
      continue;
    }
    const int K = role == ptc::ROLE_J ? J : H;
    const int Kp = role == ptc::ROLE_J ? Jp : Hp;
    // weight element (tile row mm, k); 0 outside the model
    auto wel = [&](int mm, int k) -> float {
      if (k >= K) return 0.0f;
      if (role == ptc::ROLE_J) {
        const int n = 128 * t + mm;
        if (n < V1) return w[bse + 2][(size_t)k * V1 + n];
        if (n < V1 + D) return w[bse + 3][(size_t)k * D + (n - V1)];
        return 0.0f;
      }
      if (role == ptc::ROLE_P) {
        const int j = 128 * t + mm;
        return j < J ? w[bse + 1][(size_t)k * J + j] : 0.0f;
      }
      const int u = lstm ? 32 * t + (mm >> 2) : 128 * t + mm;  // unit-major: row = 4*unit + gate
      const int g = lstm ? (mm & 3) : 0;
      if (u >= H) return 0.0f;
      const std::vector<float>& W = role == ptc::ROLE_R ? w[2 + 3 * l] : w[1 + 3 * l];
      return W[(size_t)k * (lstm ? 4 * H : H) + g * H + u];
    };
    float amax = 0.0f;
    for (int mm = 0; mm < 128; ++mm)
      for (int k = 0; k < K; ++k) amax = std::max(amax, std::fabs(wel(mm, k)));
    // scale by 2^s so max |W'| lies in [2^11, 2^12): W_lo' stays a normal fp16
    int sexp = 0;
    if (amax > 0.0f) {
      int e;
      std::frexp(amax, &e);  // amax = f * 2^e, f in [0.5, 1)
      sexp = 12 - e;
    }
    const float scale = std::ldexp(1.0f, sexp), inv = std::ldexp(1.0f, -sexp);
    int invbits;
    std::memcpy(&invbits, &inv, 4);
    roles[c].w = invbits;
    unsigned char* hi = img.data() + (size_t)c * wstride;
    uint32_t* lo = reinterpret_cast<uint32_t*>(hi + wtoff);
    const int kcr = Kp / 64, nlo = ptc::nlo_chunks(kcr);
    for (int mm = 0; mm < 128; ++mm) {
      for (int k = 0; k < Kp; ++k) row[k] = wel(mm, k) * scale;
      for (int k = 0; k < Kp; k += 2) {
        // smem image <- W_hi and TMEM pairs <- W_lo (ptc::SWAP_HILO: the reverse)
        uint16_t lb[2], sb[2];
        for (int j = 0; j < 2; ++j) {
          const float v = row[k + j];
          uint16_t hb = f2h_bits(v);
          uint16_t l = f2h_bits(v - h2f(hb));
          if (ptc::SWAP_HILO) std::swap(hb, l);
          lb[j] = l;
          sb[j] = hb;
          std::memcpy(hi + (size_t)((k + j) / 64) * 16384 + ptc::swz(mm, (k + j) % 64), &hb, 2);
        }
        lo[(size_t)(k / 2) * 128 + mm] = (uint32_t)lb[0] | ((uint32_t)lb[1] << 16);
        if (k / 64 < nlo)  // this chunk's smem-image half is TMEM-resident too
          lo[(size_t)(kcr * 32 + k / 2) * 128 + mm] = (uint32_t)sb[0] | ((uint32_t)sb[1] << 16);
      }
    }
  }
  ptc::TParams& tp = d->tp;
  tp = ptc::TParams{};
  tp.G = G;
  tp.B = d->B;
  tp.T = d->T;
  tp.ms = d->ms;
  tp.cap = d->st.cap;
  tp.algo = d->algo;
  tp.L = L;
  tp.cell = M.cell;
  tp.H = H;
  tp.Hp = Hp;
  tp.J = J;
  tp.Jp = Jp;
  tp.V1 = V1;
  tp.D = D;
  tp.NJ = NJ;
  tp.GH = M.GH;
  tp.Gg = M.G;
  tp.max_iters = d->st.max_iters;
  tp.ngrp = ngrp;
  tp.split0 = split0;
  tp.ninst = ninst;
  for (int i = 0; i <= ninst; ++i) {
    tp.ic0[i] = ic0[i];
    tp.ig0[i] = ngrp * i / ninst;  // the instances' row groups
  }
  for (int g = 0; g <= ngrp; ++g) tp.gr0[g] = (int)((long long)d->B * g / ngrp);
  for (int i = 0; i < D; ++i) tp.durations[i] = dd.durations[i];
  int4* droles = nullptr;
  CK(upload(d->mem, &droles, roles));
  tp.roles = droles;
  unsigned char* dimg = nullptr;
  CK(upload(d->mem, &dimg, img));
  tp.wimg = dimg;
  tp.wstride = wstride;
  tp.wtoff = wtoff;
  for (int l = 0; l < L; ++l) {
    float* db = nullptr;
    CK(upload(d->mem, &db, w[3 + 3 * l]));
    tp.bias[l] = db;
  }
  tp.table0 = M.table0;
  tp.fp = d->st.fp;
  tp.out_len = d->len_dev;
  for (int b = 0; b <= ptc::TRUNK; ++b) {
    if (b < L || b == ptc::TRUNK) {
      const int kc = (b == ptc::TRUNK ? Jp : Hp) / 64;
      tp.act_kc[b] = kc;
      CK(d->mem.alloc(&tp.act[b], (size_t)ngrp * 2 * kc * ptc::CHUNK));
      for (int c = 0; c < kc; ++c) {
        int n = 0;
        if (b == ptc::TRUNK) {
          n = 1;  // P tile c/2
        } else if (lstm) {
          for (int t = 0; t < NG; ++t)
            if (32 * t < 64 * (c + 1) && 32 * t + 32 > 64 * c) ++n;
        } else {
          n = 1;
        }
        tp.nprod[b][c] = n;
      }
    }
  }
  // activation tensor maps: [2 parity x 64 rows][Kp] fp16, row-major
  {
    PFN_encodeTiled enc = get_encode_tiled();
    if (!enc) return fail(RNNTG_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    for (int b = 0; b <= ptc::TRUNK; ++b) {
      if (!(b < L || b == ptc::TRUNK)) continue;
      const int Kp = tp.act_kc[b] * 64;
      const cuuint64_t dims[2] = {(cuuint64_t)Kp, (cuuint64_t)128 * ngrp};
      const cuuint64_t strides[1] = {(cuuint64_t)Kp * 2};
      const cuuint32_t estr[2] = {1, 1};
      const cuuint32_t lbox[2] = {64, 64};
      if (enc(&tp.ldmap[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, tp.act[b], dims, strides, lbox, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return fail(RNNTG_E_CUDA, "activation load tensor map");
      const bool half_tiles = lstm && b < L;  // LSTM tiles publish 32-unit boxes
      const cuuint32_t sbox[2] = {half_tiles ? 32u : 64u, 64};
      if (enc(&tp.stmap[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, tp.act[b], dims, strides, sbox, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, half_tiles ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return fail(RNNTG_E_CUDA, "activation store tensor map");
    }
  }
  for (int l = 0; l < L; ++l) CK(d->mem.alloc(&tp.hh[l], (size_t)ngrp * 2 * 64 * 32 * 128));
  d->tpw_bytes = (size_t)ngrp * ptc::NSLOT * 2 * NJ * 32 * sizeof(unsigned long long);
  CK(d->mem.alloc(&tp.pw, (size_t)ngrp * ptc::NSLOT * 2 * NJ * 32));
  CK(d->mem.alloc(&tp.ps, (size_t)ngrp * ptc::NSLOT * NJ * 32));
  // per group: counters, then the G per-CTA ack words: zeroed together before every launch
  const size_t ncnt = (size_t)ngrp * ptc::NCOUNTERS * ptc::CSTRIDE;
  d->tcnt_bytes = (ncnt + (size_t)ngrp * G) * sizeof(unsigned);
  CK(d->mem.alloc(&d->tcnt, ncnt + (size_t)ngrp * G));
  tp.cnt = d->tcnt;
  tp.ack = d->tcnt + ncnt;
  if (ngrp > 1) CK(d->mem.alloc(&tp.gst, (size_t)ngrp * G * ptc::NSV * ptc::NEPI));
  tp.tokens = d->st.tokens;
  tp.frames = d->st.frames;
  tp.scores = d->st.scores;
  tp.durs = d->st.durs;
  tp.counts = d->st.counts;
  tp.ctrl = d->st.ctrl;
  for (int r = 0; r < ptc::NROLES; ++r) tp.prof_first[r] = -1;
  for (int c = G - 1; c >= 0; --c) tp.prof_first[roles[c].x] = c;
  for (int c = 0; c < G; ++c)  // the traced I CTA: the first one with an MMA (layer 1)
    if (roles[c].x == ptc::ROLE_I && (roles[c].y & 0xff) == 1) { tp.prof_first[ptc::ROLE_I] = c; break; }
  if (env_flag("RNNTG_STAMPS", false)) CK(d->mem.alloc(&tp.stamps, (size_t)64 * G * 16));
  if (env_flag("RNNTG_PROF", false)) {
    CK(d->mem.alloc(&tp.prof, (size_t)(2 * ptc::NEV + G) * ptc::PROF_WIN));
  }
  return RNNTG_OK;
}

cudaError_t launch_tc(rnntg_decoder* d, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(d->tcnt, 0, d->tcnt_bytes, st);
  if (e != cudaSuccess) return e;
  // tagged argmax words carry step tags: clear them so a stale word from the
  // previous decode can never validate
  if ((e = cudaMemsetAsync(d->tp.pw, 0, d->tpw_bytes, st)) != cudaSuccess) return e;
  // instances add their totals into the control block
  if (d->tp.ninst > 1 && (e = cudaMemsetAsync(d->st.ctrl, 0, sizeof(Ctrl), st)) != cudaSuccess) return e;
  void* args[1] = {&d->tp};
  // the traced instantiation only when the event trace is on (RNNTG_PROF)
  const void* k = tc_kernel_for(d->tp.algo, d->tp.cell, d->tp.prof != nullptr);
  return cudaLaunchCooperativeKernel(k, dim3(d->tp.G), dim3(ptc::NTH), args, d->tsmem, st);
}

// ---------------------------------------------------------------- K6 step launches
// The graph and host-loop executors run the tensor-core kernel one decision
// per launch (STEP_ONE) after one P0 launch (STEP_INIT): the same role CTAs
// and arithmetic as K6, with the replicated control state and the
// per-thread cell / gp state kept in global memory between launches, and
// the loop flags set from the device (cudaGraphSetConditional) or read back
// by the host loop.
rnntg_status setup_tc_steps(rnntg_decoder* d, bool use_cond) {
  rnntg_status st = setup_tc(d, false);  // (one instance: the loop flags read one CTA's state)
  if (st) return st;
  ptc::TParams& tp = d->tp;
  CK(d->mem.alloc(&tp.ctl, (size_t)tp.G * ptc::CTL_INTS));
  if (!tp.gst) CK(d->mem.alloc(&tp.gst, (size_t)tp.ngrp * tp.G * ptc::NSV * ptc::NEPI));
  for (int i = 0; i < 2; ++i) {
    d->tp_step[i] = tp;
    d->tp_step[i].step_mode = i == 0 ? ptc::STEP_INIT : ptc::STEP_ONE;
    d->tp_step[i].use_cond = use_cond ? 1 : 0;
    // graph bodies run up to RNNTG_GRAPH_STEPS (default 16) decisions per
    // launch -- the WHILE body unrolled, amortising the per-launch weight
    // reload and the conditional-node relaunch (~5 us) over the decisions;
    // the sync-requiring host loop stays at one decision (and one flag
    // read-back) per launch
    const char* gs = getenv("RNNTG_GRAPH_STEPS");
    d->tp_step[i].steps_per_launch = use_cond ? std::max(1, gs ? atoi(gs) : 16) : 1;
    d->tp_step[i].pdl = use_cond && env_flag("RNNTG_GRAPH_PDL", false) ? 1 : 0;
  }
  d->tc_steps = true;
  return RNNTG_OK;
}

cudaError_t coop_node(cudaGraphNode_t n) {
  // (RNNTG_GRAPH_COOP=0: plain kernel nodes -- every CTA is resident anyway,
  // one per SM, G <= SMs, and the graph runs its nodes in order)
  if (!env_flag("RNNTG_GRAPH_COOP", true)) return cudaSuccess;
  cudaLaunchAttributeValue v{};
  v.cooperative = 1;
  return cudaGraphKernelNodeSetAttribute(n, cudaLaunchAttributeCooperative, &v);
}

cudaError_t memset_node(Builder& b, void* dst, size_t bytes) {
  cudaMemsetParams p{};
  p.dst = dst;
  p.value = 0;
  p.elementSize = 4;
  p.width = bytes / 4;
  p.height = 1;
  cudaGraphNode_t n;
  cudaError_t e = cudaGraphAddMemsetNode(&n, b.g, b.last ? &b.last : nullptr, b.last ? 1 : 0, &p);
  if (e != cudaSuccess) return e;
  b.last = n;
  b.last_kernel = false;
  return cudaSuccess;
}

// graph: counters/words reset -> K1 -> P0 launch ->
//   WHILE any live { step ; WHILE inner { step } }
// (frame-looping: the inner WHILE runs the rest of a frame's symbols;
// label-looping: it runs the blank-skipping joint steps until a row accepts)
cudaError_t build_graph_tc(rnntg_decoder* d) {
  cudaError_t e;
  if ((e = cudaGraphCreate(&d->graph, 0)) != cudaSuccess) return e;
  cudaGraphConditionalHandle ho, hi;
  if ((e = cudaGraphConditionalHandleCreate(&ho, d->graph, 0, 0)) != cudaSuccess) return e;
  if ((e = cudaGraphConditionalHandleCreate(&hi, d->graph, 0, 0)) != cudaSuccess) return e;
  for (int i = 0; i < 2; ++i) {
    d->tp_step[i].h_outer = ho;
    d->tp_step[i].h_inner = hi;
  }
  const void* k = tc_kernel_for(d->algo, d->m->dm.cell, false);
  void* a_init[1] = {&d->tp_step[0]};
  void* a_step[1] = {&d->tp_step[1]};
  const dim3 grid(d->tp.G), block(ptc::NTH);
  Builder root{d->graph};
  root.pdl = false;  // the step kernel does not wait on griddepcontrol
  if ((e = memset_node(root, d->tcnt, d->tcnt_bytes)) != cudaSuccess) return e;
  if ((e = memset_node(root, d->tp.pw, d->tpw_bytes)) != cudaSuccess) return e;
  if ((e = add_encproj(root, d)) != cudaSuccess) return e;
  if ((e = root.kernel(k, grid, block, d->tsmem, a_init)) != cudaSuccess) return e;
  if ((e = coop_node(root.last)) != cudaSuccess) return e;
  cudaGraph_t outer_body, inner_body;
  if ((e = root.while_node(ho, &outer_body)) != cudaSuccess) return e;
  Builder ob{outer_body};
  ob.pdl = false;
  if ((e = ob.kernel(k, grid, block, d->tsmem, a_step)) != cudaSuccess) return e;
  if ((e = coop_node(ob.last)) != cudaSuccess) return e;
  if ((e = ob.while_node(hi, &inner_body)) != cudaSuccess) return e;
  Builder ib{inner_body};
  if (d->tp_step[1].pdl) {
    // two step launches per inner iteration, the second a programmatic
    // dependent of the first (its CTAs load their weights while the first
    // finishes); plain kernel nodes (PDL + cooperative do not mix)
    ib.pdl = true;
    if ((e = ib.kernel(k, grid, block, d->tsmem, a_step)) != cudaSuccess) return e;
    if ((e = ib.kernel(k, grid, block, d->tsmem, a_step)) != cudaSuccess) return e;
  } else {
    ib.pdl = false;
    if ((e = ib.kernel(k, grid, block, d->tsmem, a_step)) != cudaSuccess) return e;
    if ((e = coop_node(ib.last)) != cudaSuccess) return e;
  }
  return cudaGraphInstantiate(&d->gexec, d->graph, 0);
}

cudaError_t launch_tc_step(rnntg_decoder* d, int i) {
  void* args[1] = {&d->tp_step[i]};
  return cudaLaunchCooperativeKernel(tc_kernel_for(d->algo, d->m->dm.cell, false), dim3(d->tp.G), dim3(ptc::NTH),
                                     args, d->tsmem, d->stream);
}

// ---------------------------------------------------------------- host loop
// The sync-requiring baseline (greedy_decode_baseline, decoders.cpp:546-563;
// Algorithm 1 of the paper): the SAME kernels as the graph executor, launched
// one by one from a host loop that copies the loop flags back and
// synchronises after every joint step (and every frame / outer round), i.e.
// the host round trips the conditional WHILE nodes remove.  The contrast row
// for the GPU idle fraction; rnntg_launch returns when the decode is done.
rnntg_status run_hostloop(rnntg_decoder* d) {
  const DevModel& M = d->m->dm;
  DevState s = d->st;
  s.use_cond = 0;
  cudaStream_t st = d->stream;
  const int nrb = s.nrb;
  Ctrl* hc = d->hctrl;
  auto pred = [&]() -> cudaError_t {
    if (M.cell == RNNTG_CELL_SCRIPTED) {
      ++d->n_launches;
      scripted_pred_kernel<<<1, NT, 0, st>>>(M, s);
      return cudaGetLastError();
    }
    d->n_launches += M.L + 1;
    for (int l = 0; l < M.L; ++l) {
      if (M.cell == RNNTG_CELL_LSTM)
        pred_layer_kernel<1><<<dim3(M.GH / CT, nrb), NT, layer_smem(M, l), st>>>(M, s, l);
      else
        pred_layer_kernel<0><<<dim3(M.GH / CT, nrb), NT, layer_smem(M, l), st>>>(M, s, l);
    }
    pred_proj_kernel<<<dim3(M.Jp / CT, nrb), NT, pp_smem(M), st>>>(M, s);
    return cudaGetLastError();
  };
  auto joint = [&]() -> cudaError_t {
    ++d->n_launches;
    joint_kernel<<<dim3(M.NCHT, nrb), NT, joint_smem(M), st>>>(M, s);
    return cudaGetLastError();
  };
  auto flags = [&]() -> cudaError_t {  // the per-step device -> host sync
    ++d->n_syncs;
    cudaError_t e = cudaMemcpyAsync(hc, s.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st);
    return e != cudaSuccess ? e : cudaStreamSynchronize(st);
  };
  if (M.cell != RNNTG_CELL_SCRIPTED) CK(encproj_launch(d->enc, st));
  d->n_launches += 2;
  prologue_kernel<<<148, 256, 0, st>>>(M, s);
  CK(cudaGetLastError());
  CK(pred());  // P0 = pred(blank, 0)
  CK(flags());
  if (d->algo == RNNTG_ALGO_FRAME_SYNC) {
    while (hc->t < hc->max_len && !hc->abort) {
      do {  // inner: joint + prediction, until every row blanked or sym == ms
        CK(joint());
        CK(pred());
        CK(flags());
      } while (hc->any && !hc->abort);
      ++d->n_launches;
      frame_tail_kernel<<<1, 256, 0, st>>>(M, s);
      CK(cudaGetLastError());
      CK(flags());
    }
  } else {
    while (hc->any && !hc->abort) {  // outer: any row active
      do {  // inner: joint-only blank skipping while a row needs a decision
        CK(joint());
        CK(flags());
      } while (hc->any && !hc->abort);
      CK(pred());  // acceptors' prediction step + round tail (sets `any`)
      CK(flags());
    }
  }
  return RNNTG_OK;
}

// The sync-requiring baseline on the tensor-core step kernel: the same
// launches as the graph executor's loop bodies, issued by the host, with the
// loop flags copied back and synchronised after every step.
rnntg_status run_hostloop_tc(rnntg_decoder* d) {
  cudaStream_t st = d->stream;
  Ctrl* hc = d->hctrl;
  auto flags = [&]() -> cudaError_t {
    ++d->n_syncs;
    cudaError_t e = cudaMemcpyAsync(hc, d->st.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st);
    return e != cudaSuccess ? e : cudaStreamSynchronize(st);
  };
  CK(cudaMemsetAsync(d->tcnt, 0, d->tcnt_bytes, st));
  CK(cudaMemsetAsync(d->tp.pw, 0, d->tpw_bytes, st));
  CK(encproj_launch(d->enc, st));
  CK(launch_tc_step(d, 0));  // P0
  d->n_launches += 2;
  CK(flags());
  while (hc->any && !hc->err) {
    do {  // inner: frame-looping -- the frame's symbols; label-looping -- blank skipping
      CK(launch_tc_step(d, 1));
      ++d->n_launches;
      CK(flags());
    } while (hc->any && hc->abort && !hc->err);
  }
  return RNNTG_OK;
}

cudaError_t build_graph(rnntg_decoder* d) {
  const bool pdl = env_flag("RNNTG_PDL", true);
  cudaError_t e;
  if ((e = cudaGraphCreate(&d->graph, 0)) != cudaSuccess) return e;
  if ((e = cudaGraphConditionalHandleCreate(&d->st.h_outer, d->graph, 0, 0)) != cudaSuccess)
    return e;
  if ((e = cudaGraphConditionalHandleCreate(&d->st.h_inner, d->graph, 0, 0)) != cudaSuccess)
    return e;
  d->st.use_cond = 1;
  d->arg_m = d->m->dm;
  d->arg_s = d->st;
  for (int l = 0; l < MAXL; ++l) d->arg_l[l] = l;

  Builder root{d->graph};
  root.pdl = pdl;
  if (d->m->dm.cell != RNNTG_CELL_SCRIPTED && (e = add_encproj(root, d)) != cudaSuccess) return e;
  {
    void* args[2] = {&d->arg_m, &d->arg_s};
    if ((e = root.kernel((const void*)prologue_kernel, dim3(148), dim3(256), 0, args)) !=
        cudaSuccess)
      return e;
  }
  if ((e = add_pred_step(root, d)) != cudaSuccess) return e;  // P0 = pred(blank, 0)
  cudaGraph_t outer_body;
  if ((e = root.while_node(d->st.h_outer, &outer_body)) != cudaSuccess) return e;
  Builder ob{outer_body};
  ob.pdl = pdl;
  cudaGraph_t inner_body;
  if ((e = ob.while_node(d->st.h_inner, &inner_body)) != cudaSuccess) return e;
  Builder ib{inner_body};
  ib.pdl = pdl;
  if (d->algo == RNNTG_ALGO_FRAME_SYNC) {
    // WHILE t < max_len { WHILE any(!blank) && sym < ms { joint; pred } ; tail }
    if ((e = add_joint(ib, d)) != cudaSuccess) return e;
    if ((e = add_pred_step(ib, d)) != cudaSuccess) return e;
    void* args[2] = {&d->arg_m, &d->arg_s};
    if ((e = ob.kernel((const void*)frame_tail_kernel, dim3(1), dim3(256), 0, args)) !=
        cudaSuccess)
      return e;
  } else {
    // WHILE any(active) { WHILE any(need) { joint } ; pred (accepted rows) }
    if ((e = add_joint(ib, d)) != cudaSuccess) return e;
    if ((e = add_pred_step(ob, d)) != cudaSuccess) return e;
  }
  return cudaGraphInstantiate(&d->gexec, d->graph, 0);
}

}  // namespace

// =====================================================================
extern "C" {

const char* rnntg_last_error(void) { return g_err.c_str(); }
int rnntg_abi_version(void) { return RNNTG_ABI_VERSION; }

int rnntg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

rnntg_status rnntg_model_create(int device, const rnntg_dims* dims, const float* const* weights,
                                int nweights, rnntg_model** out) {
  if (!out) return fail(RNNTG_E_VALUE, "out is null");
  *out = nullptr;
  rnntg_status st = validate_dims(dims);
  if (st) return st;
  if (!weights || nweights != num_weights(dims))
    return fail(RNNTG_E_VALUE, "expected " + std::to_string(num_weights(dims)) + " weight tensors");
  for (int i = 0; i < nweights; ++i)
    if (!weights[i]) return fail(RNNTG_E_VALUE, "null weight pointer");
  if (rnntg_device_count() == 0) return fail(RNNTG_E_CUDA, "no CUDA device");
  CK(cudaSetDevice(device));
  auto* m = new rnntg_model;
  m->device = device;
  m->dims = *dims;
  DevModel& M = m->dm;
  const rnntg_dims& d = *dims;
  M.V1 = d.vocab + 1;
  M.E = d.embed;
  M.H = d.hidden;
  M.Hp = round_up(d.hidden, 64);
  M.L = d.layers;
  M.cell = d.cell;
  M.G = d.cell == RNNTG_CELL_LSTM ? 4 : 1;
  M.GH = M.G * M.Hp;
  M.J = d.joint;
  M.Jp = round_up(d.joint, 64);
  M.F = d.feature;
  M.Fp = round_up(d.feature, 64);
  M.D = d.num_durations;
  for (int i = 0; i < M.D; ++i) M.durations[i] = d.durations[i];
  M.V1p = round_up(M.V1, CT);
  M.NOUT = M.V1p + (M.D ? CT : 0);
  M.NCH = M.V1p / CT;
  M.NCHT = M.NCH + (M.D ? 1 : 0);
  const int H = M.H, Hp = M.Hp, G = M.G, GH = M.GH, J = M.J, Jp = M.Jp, V1 = M.V1;
  auto fail_free = [&](rnntg_status s, const std::string& msg) {
    m->mem.release();
    delete m;
    return fail(s, msg);
  };
#define CKM(expr)                                                                   \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail_free(RNNTG_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)
  // gate-column interleave: reference column g*H + u -> u*G + g
  auto gcol = [&](int refcol) { return (refcol % H) * G + refcol / H; };
  const int gcols = G * H;
  for (int l = 0; l < M.L; ++l) {
    const float* w_ih = weights[1 + 3 * l];
    const float* w_hh = weights[2 + 3 * l];
    const float* bias = weights[3 + 3 * l];
    const int rows = l == 0 ? Hp : 2 * Hp;
    std::vector<float> W((size_t)rows * GH, 0.0f);
    const int hh_row0 = l == 0 ? 0 : Hp;
    for (int k = 0; k < H; ++k)
      for (int c = 0; c < gcols; ++c) W[(size_t)(hh_row0 + k) * GH + gcol(c)] = w_hh[(size_t)k * gcols + c];
    if (l > 0)
      for (int k = 0; k < H; ++k)
        for (int c = 0; c < gcols; ++c) W[(size_t)k * GH + gcol(c)] = w_ih[(size_t)k * gcols + c];
    float* dw = nullptr;
    CKM(upload(m->mem, &dw, tile16(W, rows, GH)));
    M.w[l] = dw;
    std::vector<float> bv(GH, 0.0f);
    for (int c = 0; c < gcols; ++c) bv[gcol(c)] = bias[c];
    float* db = nullptr;
    CKM(upload(m->mem, &db, bv));
    M.bias[l] = db;
  }
  {  // table0 = embedding @ W_ih0 (exact sequential k, on device)
    std::vector<float> emb(weights[0], weights[0] + (size_t)V1 * M.E);
    std::vector<float> wih(weights[1], weights[1] + (size_t)M.E * gcols);
    float *demb = nullptr, *dwih = nullptr, *dtab = nullptr;
    CKM(upload(m->mem, &demb, emb));
    CKM(upload(m->mem, &dwih, wih));
    CKM(m->mem.alloc(&dtab, (size_t)V1 * GH));
    table0_kernel<<<dim3((gcols + 127) / 128, V1), 128>>>(demb, dwih, dtab, V1, M.E, gcols, G, H,
                                                          Hp);
    CKM(cudaGetLastError());
    CKM(cudaDeviceSynchronize());
    M.table0 = dtab;
  }
  const int base = 1 + 3 * M.L;
  {
    std::vector<float> pp((size_t)Hp * Jp, 0.0f);
    for (int k = 0; k < H; ++k)
      for (int j = 0; j < J; ++j) pp[(size_t)k * Jp + j] = weights[base + 1][(size_t)k * J + j];
    float* dp = nullptr;
    CKM(upload(m->mem, &dp, tile16(pp, Hp, Jp)));
    M.pred_proj = dp;
  }
  {
    std::vector<float> oe((size_t)Jp * M.NOUT, 0.0f);
    for (int k = 0; k < J; ++k) {
      for (int v = 0; v < V1; ++v) oe[(size_t)k * M.NOUT + v] = weights[base + 2][(size_t)k * V1 + v];
      for (int c = 0; c < M.D; ++c)
        oe[(size_t)k * M.NOUT + M.V1p + c] = weights[base + 3][(size_t)k * M.D + c];
    }
    float* dp = nullptr;
    CKM(upload(m->mem, &dp, tile16(oe, Jp, M.NOUT)));
    M.out_ext = dp;
  }
  {
    std::vector<float> en((size_t)M.Fp * Jp, 0.0f);
    for (int k = 0; k < M.F; ++k)
      for (int j = 0; j < J; ++j) en[(size_t)k * Jp + j] = weights[base][(size_t)k * J + j];
    float* dp = nullptr;
    CKM(upload(m->mem, &dp, en));
    M.enc = dp;
    // tcgen05 operands: enc^T K-major [Jp][Fp], split into tf32 hi / lo
    std::vector<float> hi((size_t)Jp * M.Fp, 0.0f), lo((size_t)Jp * M.Fp, 0.0f);
    for (int k = 0; k < M.F; ++k)
      for (int j = 0; j < J; ++j) {
        const float v = weights[base][(size_t)k * J + j];
        float h;
        uint32_t u;
        std::memcpy(&u, &v, 4);
        u &= 0xffffe000u;
        std::memcpy(&h, &u, 4);
        hi[(size_t)j * M.Fp + k] = h;
        lo[(size_t)j * M.Fp + k] = v - h;
      }
    float *dh = nullptr, *dl = nullptr;
    CKM(upload(m->mem, &dh, hi));
    CKM(upload(m->mem, &dl, lo));
    M.enc_hi = dh;
    M.enc_lo = dl;
  }
  CKM(set_smem_attrs(M));
  m->tc_ok = encproj_tc_supported(M);
  if (!m->tc_ok)
    return fail_free(RNNTG_E_CUDA,
                     "tcgen05 encoder projection unavailable (needs an sm_100 B200 device)");
  {
    m->host_w.resize(nweights);
    const rnntg_dims& dd = *dims;
    const int V1_ = dd.vocab + 1, Gc = dd.cell == RNNTG_CELL_LSTM ? 4 * dd.hidden : dd.hidden;
    for (int l = 0; l < dd.layers; ++l) {
      const int in = l == 0 ? dd.embed : dd.hidden;
      m->host_w[1 + 3 * l].assign(weights[1 + 3 * l], weights[1 + 3 * l] + (size_t)in * Gc);
      m->host_w[2 + 3 * l].assign(weights[2 + 3 * l], weights[2 + 3 * l] + (size_t)dd.hidden * Gc);
      m->host_w[3 + 3 * l].assign(weights[3 + 3 * l], weights[3 + 3 * l] + Gc);
    }
    const int bse = 1 + 3 * dd.layers;
    m->host_w[bse + 1].assign(weights[bse + 1], weights[bse + 1] + (size_t)dd.hidden * dd.joint);
    m->host_w[bse + 2].assign(weights[bse + 2], weights[bse + 2] + (size_t)dd.joint * V1_);
    if (dd.num_durations)
      m->host_w[bse + 3].assign(weights[bse + 3],
                                weights[bse + 3] + (size_t)dd.joint * dd.num_durations);
  }
#undef CKM
  *out = m;
  return RNNTG_OK;
}

rnntg_status rnntg_model_destroy(rnntg_model* m) {
  if (!m) return RNNTG_OK;
  cudaSetDevice(m->device);
  m->mem.release();
  delete m;
  return RNNTG_OK;
}

rnntg_status rnntg_model_create_scripted(int device, int vocab, int batch, int frames, int umax,
                                         const int32_t* labels, const int32_t* fs_arr,
                                         const int32_t* dur_arr, int num_durations,
                                         const int32_t* durations, const int32_t* dur_val,
                                         rnntg_model** out) {
  if (!out) return fail(RNNTG_E_VALUE, "out is null");
  *out = nullptr;
  if (vocab < 1 || batch < 1 || frames < 1 || umax < 1) return fail(RNNTG_E_VALUE, "scripted model dims must be >= 1");
  if (num_durations < 0 || num_durations > MAXD) return fail(RNNTG_E_VALUE, "bad duration class count");
  if (!labels || !fs_arr || !dur_arr || (num_durations > 0 && (!durations || !dur_val)))
    return fail(RNNTG_E_VALUE, "null scripted table");
  if (rnntg_device_count() == 0) return fail(RNNTG_E_CUDA, "no CUDA device");
  CK(cudaSetDevice(device));
  auto* m = new rnntg_model;
  m->device = device;
  rnntg_dims& dd = m->dims;
  dd = rnntg_dims{};
  dd.vocab = vocab;
  dd.embed = dd.hidden = dd.joint = 1;
  dd.layers = 1;
  dd.cell = RNNTG_CELL_SCRIPTED;
  dd.feature = 2;  // (utterance, frame) features, ScriptedModel::make_features
  dd.num_durations = num_durations;
  for (int i = 0; i < num_durations; ++i) dd.durations[i] = durations[i];
  DevModel& M = m->dm;
  M = DevModel{};
  M.V1 = vocab + 1;
  M.E = M.H = M.J = 1;
  M.Hp = M.Jp = 64;
  M.L = 1;
  M.cell = RNNTG_CELL_SCRIPTED;
  M.G = 1;
  M.GH = M.Hp;
  M.F = 2;
  M.Fp = 64;
  M.D = num_durations;
  for (int i = 0; i < M.D; ++i) M.durations[i] = durations[i];
  M.V1p = round_up(M.V1, CT);
  M.NOUT = M.V1p + (M.D ? CT : 0);
  M.NCH = M.V1p / CT;
  M.NCHT = M.NCH + (M.D ? 1 : 0);
  M.s_B = batch;
  M.s_T = frames;
  M.s_U = umax;
  const size_t nl = (size_t)batch * frames * umax, nf = (size_t)batch * (frames + 1), nd = (size_t)batch * frames;
  std::vector<int32_t> dv((size_t)batch * frames * (umax + 1), 1);
  if (num_durations > 0) std::memcpy(dv.data(), dur_val, dv.size() * sizeof(int32_t));
  int *dl = nullptr, *df = nullptr, *da = nullptr, *dvd = nullptr;
  cudaError_t e;
  if ((e = m->mem.alloc(&dl, nl)) != cudaSuccess || (e = m->mem.alloc(&df, nf)) != cudaSuccess ||
      (e = m->mem.alloc(&da, nd)) != cudaSuccess || (e = m->mem.alloc(&dvd, dv.size())) != cudaSuccess ||
      (e = cudaMemcpy(dl, labels, nl * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(df, fs_arr, nf * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(da, dur_arr, nd * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(dvd, dv.data(), dv.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess) {
    m->mem.release();
    delete m;
    return fail(RNNTG_E_CUDA, std::string("scripted model upload: ") + cudaGetErrorString(e));
  }
  M.s_lab = dl;
  M.s_fsarr = df;
  M.s_darr = da;
  M.s_dval = dvd;
  *out = m;
  return RNNTG_OK;
}

rnntg_status rnntg_decoder_create(rnntg_model* m, int algo, int exec, int batch, int max_frames,
                                  int max_symbols, rnntg_decoder** out) {
  if (!out) return fail(RNNTG_E_VALUE, "out is null");
  *out = nullptr;
  if (!m) return fail(RNNTG_E_STATE, "model is null");
  if (batch < 1 || max_frames < 1) return fail(RNNTG_E_VALUE, "batch and frames must be >= 1");
  if (max_symbols < 1) return fail(RNNTG_E_VALUE, "max_symbols must be >= 1");
  if (batch > RB * MAXRB) return fail(RNNTG_E_VALUE, "batch must be <= 1024 per decoder");
  if (algo < 0 || algo > 2) return fail(RNNTG_E_VALUE, "unknown algo");
  if (algo == RNNTG_ALGO_TDT_LABEL_LOOP && m->dm.D == 0)
    return fail(RNNTG_E_STATE, "duration-head decoding needs a model with a duration head");
  if (exec < RNNTG_EXEC_GRAPH || exec > RNNTG_EXEC_GRAPH_FFMA)
    return fail(RNNTG_E_VALUE, "unknown exec mode");
  CK(cudaSetDevice(m->device));
  if (exec == RNNTG_EXEC_TENSOR && batch > ptc::MAXB * ptc::MAXG && m->dm.cell != RNNTG_CELL_SCRIPTED) {
    // balanced sub-batches, one tensor-core decoder each, sharing one stream
    auto* d = new rnntg_decoder;
    d->m = m;
    d->algo = algo;
    d->exec = exec;
    d->B = batch;
    d->T = max_frames;
    d->ms = max_symbols;
    const int nsub = (batch + ptc::MAXB * ptc::MAXG - 1) / (ptc::MAXB * ptc::MAXG);
    cudaError_t e = cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&d->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&d->ev1);
    if (e != cudaSuccess) {
      rnntg_decoder_destroy(d);
      return fail(RNNTG_E_CUDA, std::string("decoder setup: ") + cudaGetErrorString(e));
    }
    for (int i = 0, b0 = 0; i < nsub; ++i) {
      const int bi = batch / nsub + (i < batch % nsub ? 1 : 0);
      rnntg_decoder* sd = nullptr;
      const rnntg_status st = rnntg_decoder_create(m, algo, exec, bi, max_frames, max_symbols, &sd);
      if (st) {
        rnntg_decoder_destroy(d);
        return st;
      }
      cudaStreamDestroy(sd->stream);  // run on the parent's stream, in order
      sd->stream = d->stream;
      sd->owns_stream = false;
      d->subs.push_back(sd);
      d->sub_b0.push_back(b0);
      b0 += bi;
    }
    d->st.cap = d->subs[0]->st.cap;
    *out = d;
    return RNNTG_OK;
  }
  auto* d = new rnntg_decoder;
  d->m = m;
  d->algo = algo;
  d->exec = exec;
  d->B = batch;
  d->T = max_frames;
  d->ms = max_symbols;
  rnntg_status st = alloc_state(m, d->mem, d->st, algo, batch, max_frames, max_symbols, false);
  cudaError_t e = cudaSuccess;
  if (!st) {
    if ((e = d->mem.alloc(&d->x_dev, (size_t)batch * max_frames * m->dm.Fp)) == cudaSuccess &&
        (e = d->mem.alloc(&d->len_dev, (size_t)batch)) == cudaSuccess &&
        (e = d->mem.alloc(&d->len_bad, (size_t)1)) == cudaSuccess &&
        (e = cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking)) == cudaSuccess &&
        (e = cudaEventCreate(&d->ev0)) == cudaSuccess &&
        (e = cudaEventCreate(&d->ev1)) == cudaSuccess) {
      d->st.x = d->x_dev;
      d->st.out_len = d->len_dev;
      if (m->dm.cell == RNNTG_CELL_SCRIPTED && exec != RNNTG_EXEC_GRAPH && exec != RNNTG_EXEC_HOSTLOOP &&
          exec != RNNTG_EXEC_GRAPH_FFMA)
        st = fail(RNNTG_E_VALUE, "scripted models run on the graph or host-loop executor");
      else if (m->dm.cell != RNNTG_CELL_SCRIPTED &&
               !encproj_plan(d->enc, m->dm, d->x_dev, d->st.fp, batch * max_frames))
        st = fail(RNNTG_E_CUDA, "cannot encode TMA tensor maps for the encoder projection");
      else if (exec == RNNTG_EXEC_GRAPH || exec == RNNTG_EXEC_HOSTLOOP) {
        // the tensor-core step kernel when the shape fits it; else the FFMA step kernels
        const bool tc = m->dm.cell != RNNTG_CELL_SCRIPTED && env_flag("RNNTG_TC_STEPS", true) &&
                        setup_tc_steps(d, exec == RNNTG_EXEC_GRAPH) == RNNTG_OK;
        if (exec == RNNTG_EXEC_HOSTLOOP) e = cudaMallocHost(&d->hctrl, sizeof(Ctrl));
        else e = tc ? build_graph_tc(d) : build_graph(d);
      } else if (exec == RNNTG_EXEC_GRAPH_FFMA) e = build_graph(d);
      else if (exec == RNNTG_EXEC_TENSOR) st = setup_tc(d);
      else st = setup_persistent(d);
    }
  }
  if (!st && e != cudaSuccess) st = fail(RNNTG_E_CUDA, std::string("decoder setup: ") + cudaGetErrorString(e));
  if (st) {
    rnntg_decoder_destroy(d);
    return st;
  }
  *out = d;
  return RNNTG_OK;
}

rnntg_status rnntg_decoder_destroy(rnntg_decoder* d) {
  if (!d) return RNNTG_OK;
  cudaSetDevice(d->m->device);
  if (d->stream) cudaStreamSynchronize(d->stream);
  for (rnntg_decoder* sd : d->subs) rnntg_decoder_destroy(sd);
  d->subs.clear();
  if (!d->owns_stream) d->stream = nullptr;
  if (d->gexec) cudaGraphExecDestroy(d->gexec);
  if (d->lexec) cudaGraphExecDestroy(d->lexec);
  if (d->graph) cudaGraphDestroy(d->graph);
  if (d->ev0) cudaEventDestroy(d->ev0);
  if (d->ev1) cudaEventDestroy(d->ev1);
  if (d->stream) cudaStreamDestroy(d->stream);
  if (d->hctrl) cudaFreeHost(d->hctrl);
  d->mem.release();
  delete d;
  return RNNTG_OK;
}

int rnntg_decoder_capacity(const rnntg_decoder* d) { return d ? d->st.cap : 0; }
void* rnntg_decoder_stream(rnntg_decoder* d) { return d ? (void*)d->stream : nullptr; }

static rnntg_status check_lengths(const rnntg_decoder* d, const int32_t* out_len) {
  for (int b = 0; b < d->B; ++b)
    if (out_len[b] < 0 || out_len[b] > d->T)  // decoders.cpp:136-140
      return fail(RNNTG_E_DIMENSION, "out_len entries must lie in [0, frames]");
  return RNNTG_OK;
}

rnntg_status rnntg_bind(rnntg_decoder* d, const float* x, const int32_t* out_len) {
  if (!d) return fail(RNNTG_E_STATE, "decoder is null");
  if (!x || !out_len) return fail(RNNTG_E_DIMENSION, "null input");
  rnntg_status st = check_lengths(d, out_len);
  if (st) return st;
  CK(cudaSetDevice(d->m->device));
  const size_t F = d->m->dm.F, Fp = d->m->dm.Fp;
  if (!d->subs.empty()) {
    for (size_t i = 0; i < d->subs.size(); ++i)
      if ((st = rnntg_bind(d->subs[i], x + (size_t)d->sub_b0[i] * d->T * F, out_len + d->sub_b0[i])) != RNNTG_OK)
        return st;
    d->bound = true;
    return RNNTG_OK;
  }
  CK(cudaMemcpy2DAsync(d->x_dev, Fp * sizeof(float), x, F * sizeof(float), F * sizeof(float),
                       (size_t)d->B * d->T, cudaMemcpyHostToDevice, d->stream));
  CK(cudaMemcpyAsync(d->len_dev, out_len, sizeof(int32_t) * d->B, cudaMemcpyHostToDevice,
                     d->stream));
  d->bound = true;
  return RNNTG_OK;
}

// Device-resident lengths are validated on the device, in stream order (no
// host round trip per bind): an entry outside [0, T] (decoders.cpp:136-140)
// is clamped so the decode stays in bounds, flagged, and reported as
// DimensionError by the next rnntg_sync / rnntg_read.
__global__ void check_lengths_kernel(int* len, int B, int T, int* bad) {
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int v = len[b];
    if (v < 0 || v > T) {
      len[b] = v < 0 ? 0 : T;
      atomicExch(bad, 1);
    }
  }
}

rnntg_status rnntg_bind_device(rnntg_decoder* d, const float* x_dev, const int32_t* len_dev) {
  if (!d) return fail(RNNTG_E_STATE, "decoder is null");
  if (!x_dev || !len_dev) return fail(RNNTG_E_DIMENSION, "null input");
  CK(cudaSetDevice(d->m->device));
  rnntg_status st = RNNTG_OK;
  const size_t F = d->m->dm.F, Fp = d->m->dm.Fp;
  if (!d->subs.empty()) {
    for (size_t i = 0; i < d->subs.size(); ++i)
      if ((st = rnntg_bind_device(d->subs[i], x_dev + (size_t)d->sub_b0[i] * d->T * F, len_dev + d->sub_b0[i])) !=
          RNNTG_OK)
        return st;
    d->bound = true;
    return RNNTG_OK;
  }
  CK(cudaMemcpy2DAsync(d->x_dev, Fp * sizeof(float), x_dev, F * sizeof(float), F * sizeof(float),
                       (size_t)d->B * d->T, cudaMemcpyDeviceToDevice, d->stream));
  CK(cudaMemcpyAsync(d->len_dev, len_dev, sizeof(int32_t) * d->B, cudaMemcpyDeviceToDevice,
                     d->stream));
  check_lengths_kernel<<<1, 256, 0, d->stream>>>(d->len_dev, d->B, d->T, d->len_bad);
  CK(cudaGetLastError());
  d->bound = true;
  return RNNTG_OK;
}

// issue the persistent executors' launch sequence on st
cudaError_t issue_persistent(rnntg_decoder* d, cudaStream_t st) {
  cudaError_t e = encproj_launch(d->enc, st);
  if (e != cudaSuccess) return e;
  if (d->exec == RNNTG_EXEC_TENSOR) return launch_tc(d, st);
  void* args[1] = {&d->pp};
  return cudaLaunchCooperativeKernel((const void*)pk::persistent_kernel, dim3(d->pp.G), dim3(pk::NTH), args, d->psmem,
                                     st);
}

// capture issue_persistent into d->lexec once; on any failure the direct
// launches stay in use (the capture leaves no error state behind)
void capture_persistent(rnntg_decoder* d) {
  d->ltried = true;
  if (!env_flag("RNNTG_LAUNCH_GRAPH", true)) return;
  cudaGraph_t g = nullptr;
  if (cudaStreamBeginCapture(d->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  const cudaError_t e = issue_persistent(d, d->stream);
  const cudaError_t e2 = cudaStreamEndCapture(d->stream, &g);
  if (e != cudaSuccess || e2 != cudaSuccess || !g || cudaGraphInstantiate(&d->lexec, g, 0) != cudaSuccess)
    d->lexec = nullptr;
  if (g) cudaGraphDestroy(g);
  cudaGetLastError();
}

rnntg_status rnntg_launch(rnntg_decoder* d) {
  if (!d) return fail(RNNTG_E_STATE, "decoder is null");
  if (!d->bound) return fail(RNNTG_E_STATE, "captured decoder is not initialized (no inputs bound)");
  CK(cudaSetDevice(d->m->device));
  if (!d->subs.empty()) {
    CK(cudaEventRecord(d->ev0, d->stream));
    for (rnntg_decoder* sd : d->subs) {
      const rnntg_status st = rnntg_launch(sd);
      if (st) return st;
    }
    CK(cudaEventRecord(d->ev1, d->stream));
    d->launched = true;
    return RNNTG_OK;
  }
  if ((d->exec == RNNTG_EXEC_PERSISTENT || d->exec == RNNTG_EXEC_TENSOR) && !d->ltried) capture_persistent(d);
  CK(cudaEventRecord(d->ev0, d->stream));
  d->n_syncs = d->n_graph_launches = 0;
  d->n_launches = d->exec == RNNTG_EXEC_PERSISTENT || d->exec == RNNTG_EXEC_TENSOR ? 2 : 0;
  if (d->exec == RNNTG_EXEC_GRAPH || d->exec == RNNTG_EXEC_GRAPH_FFMA) d->n_launches = d->n_graph_launches = 1;
  if (d->exec == RNNTG_EXEC_PERSISTENT || d->exec == RNNTG_EXEC_TENSOR) {
    if (d->lexec) {
      CK(cudaGraphLaunch(d->lexec, d->stream));
      d->n_graph_launches = 1;
      d->n_launches = 1;
    } else {
      CK(issue_persistent(d, d->stream));
    }
  } else if (d->exec == RNNTG_EXEC_HOSTLOOP) {
    const rnntg_status st = d->tc_steps ? run_hostloop_tc(d) : run_hostloop(d);
    if (st) return st;
  } else {
    CK(cudaGraphLaunch(d->gexec, d->stream));
  }
  CK(cudaEventRecord(d->ev1, d->stream));
  d->launched = true;
  return RNNTG_OK;
}

rnntg_status rnntg_sync(rnntg_decoder* d) {
  if (!d) return fail(RNNTG_E_STATE, "decoder is null");
  CK(cudaSetDevice(d->m->device));
  CK(cudaStreamSynchronize(d->stream));
  if (d->launched) ++d->n_syncs;
  for (rnntg_decoder* sd : d->subs) {
    const rnntg_status st = rnntg_sync(sd);
    if (st) return st;
  }
  if (!d->subs.empty()) return RNNTG_OK;
  if (d->len_bad) {  // device-bound lengths out of range (rnntg_bind_device)
    int bad = 0;
    CK(cudaMemcpy(&bad, d->len_bad, sizeof(int), cudaMemcpyDeviceToHost));
    if (bad) {
      CK(cudaMemset(d->len_bad, 0, sizeof(int)));
      return fail(RNNTG_E_DIMENSION, "out_len entries must lie in [0, frames]");
    }
  }
  if (d->launched) {
    int err = 0;
    CK(cudaMemcpy(&err, &d->st.ctrl->err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err == ERR_RUNAWAY) return fail(RNNTG_E_RUNAWAY, "while node exceeded the iteration cap");
  }
  return RNNTG_OK;
}

rnntg_status rnntg_read(rnntg_decoder* d, int32_t* counts, int32_t* tokens, int32_t* frames,
                        float* scores, int32_t* durations, int cap) {
  if (!d) return fail(RNNTG_E_STATE, "decoder is null");
  rnntg_status st = rnntg_sync(d);
  if (st) return st;
  const int B = d->B, dc = d->st.cap;
  if (cap < 1) return fail(RNNTG_E_VALUE, "cap must be >= 1");
  if (!d->subs.empty()) {
    for (size_t i = 0; i < d->subs.size(); ++i) {
      const size_t r = (size_t)d->sub_b0[i], o = r * cap;
      if ((st = rnntg_read(d->subs[i], counts ? counts + r : nullptr, tokens ? tokens + o : nullptr,
                           frames ? frames + o : nullptr, scores ? scores + o : nullptr,
                           durations ? durations + o : nullptr, cap)) != RNNTG_OK)
        return st;
    }
    return RNNTG_OK;
  }
  std::vector<int32_t> cnt(B);
  CK(cudaMemcpy(cnt.data(), d->st.counts, sizeof(int32_t) * B, cudaMemcpyDeviceToHost));
  if (counts) std::memcpy(counts, cnt.data(), sizeof(int32_t) * B);
  const int w = std::min(cap, dc);
  auto copy2d = [&](void* dst, const void* src, size_t es) -> cudaError_t {
    if (!dst) return cudaSuccess;
    return cudaMemcpy2D(dst, es * cap, src, es * dc, es * w, B, cudaMemcpyDeviceToHost);
  };
  CK(copy2d(tokens, d->st.tokens, 4));
  CK(copy2d(frames, d->st.frames, 4));
  CK(copy2d(scores, d->st.scores, 4));
  CK(copy2d(durations, d->st.durs, 4));
  return RNNTG_OK;
}

rnntg_status rnntg_host_counts(rnntg_decoder* d, int64_t* syncs, int64_t* launches, int64_t* graph_launches) {
  if (!d || !syncs || !launches || !graph_launches) return fail(RNNTG_E_STATE, "null argument");
  *syncs = d->n_syncs;
  *launches = d->n_launches;
  *graph_launches = d->n_graph_launches;
  for (rnntg_decoder* sd : d->subs) {  // sub-decoders' syncs are the parent's
    *launches += sd->n_launches;
    *graph_launches += sd->n_graph_launches;
  }
  return RNNTG_OK;
}

rnntg_status rnntg_get_stats(rnntg_decoder* d, rnntg_stats* s) {
  if (!d || !s) return fail(RNNTG_E_STATE, "null argument");
  rnntg_status st = rnntg_sync(d);
  if (st) return st;
  if (!d->subs.empty()) {  // joint evaluations etc. summed over the sub-batches
    rnntg_stats a{};
    for (rnntg_decoder* sd : d->subs) {
      rnntg_stats x{};
      if ((st = rnntg_get_stats(sd, &x)) != RNNTG_OK) return st;
      a.joint_evals += x.joint_evals;
      a.pred_steps += x.pred_steps;
      a.outer_iters += x.outer_iters;
      a.emitted += x.emitted;
    }
    if (d->launched) CK(cudaEventElapsedTime(&a.gpu_ms, d->ev0, d->ev1));
    *s = a;
    return RNNTG_OK;
  }
  Ctrl c;
  CK(cudaMemcpy(&c, d->st.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
  std::vector<int32_t> cnt(d->B);
  CK(cudaMemcpy(cnt.data(), d->st.counts, sizeof(int32_t) * d->B, cudaMemcpyDeviceToHost));
  s->joint_evals = c.joint_evals;
  s->pred_steps = c.pred_steps;
  s->outer_iters = c.outer_iters;
  s->emitted = 0;
  for (int v : cnt) s->emitted += v;
  s->gpu_ms = 0.0f;
  if (d->launched) CK(cudaEventElapsedTime(&s->gpu_ms, d->ev0, d->ev1));
  return RNNTG_OK;
}

// ---------------------------------------------------------------- step API
rnntg_status rnntg_step_joint(rnntg_model* m, int batch, const float* f, const float* g,
                              float* logp, float* dur_logp) {
  if (!m) return fail(RNNTG_E_STATE, "model is null");
  if (m->dm.cell == RNNTG_CELL_SCRIPTED) return fail(RNNTG_E_VALUE, "not available for a scripted model");
  if (batch < 1 || batch > RB * MAXRB) return fail(RNNTG_E_VALUE, "bad batch");
  if (!f || !g || !logp) return fail(RNNTG_E_DIMENSION, "null buffer");
  CK(cudaSetDevice(m->device));
  const DevModel& M = m->dm;
  DevBuf mem;
  DevState s;
  rnntg_status st = alloc_state(m, mem, s, RNNTG_ALGO_FRAME_SYNC, batch, 1, 1, true);
  if (st) {
    mem.release();
    return st;
  }
  float* xd = nullptr;
  int* lens = nullptr;
  auto run = [&]() -> rnntg_status {
    CK(mem.alloc(&xd, (size_t)batch * M.Fp));
    CK(mem.alloc(&lens, (size_t)batch));
    CK(cudaMemcpy2D(xd, sizeof(float) * M.Fp, f, sizeof(float) * M.F, sizeof(float) * M.F, batch,
                    cudaMemcpyHostToDevice));
    s.x = xd;
    s.out_len = lens;
    s.use_cond = 0;
    // encoder projection of the B single-frame rows
    EncPlan plan;
    if (!encproj_plan(plan, M, xd, s.fp, batch)) return fail(RNNTG_E_CUDA, "tensor map encode failed");
    CK(encproj_launch(plan, 0));
    // h_top' rows = g (state parity 0 -> next buffer is 1)
    CK(cudaMemcpy2D(s.h[M.L - 1][1], sizeof(float) * M.Hp, g, sizeof(float) * M.H,
                    sizeof(float) * M.H, batch, cudaMemcpyHostToDevice));
    std::vector<int> ones(batch, 1), zeros(batch, 0);
    CK(cudaMemcpy(s.accept, ones.data(), sizeof(int) * batch, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s.done, zeros.data(), sizeof(int) * batch, cudaMemcpyHostToDevice));
    CK(cudaMemset(s.ctrl, 0, sizeof(Ctrl)));
    pred_proj_kernel<<<dim3(M.Jp / CT, s.nrb), NT, pp_smem(M)>>>(M, s);
    CK(cudaGetLastError());
    joint_kernel<<<dim3(M.NCHT, s.nrb), NT, joint_smem(M)>>>(M, s);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> lg((size_t)s.Bp * M.NOUT), lse(2 * s.Bp);
    CK(cudaMemcpy(lg.data(), s.dbg_logits, sizeof(float) * lg.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(lse.data(), s.dbg_lse, sizeof(float) * lse.size(), cudaMemcpyDeviceToHost));
    for (int b = 0; b < batch; ++b) {
      for (int v = 0; v < M.V1; ++v) logp[(size_t)b * M.V1 + v] = lg[(size_t)b * M.NOUT + v] - lse[b];
      if (dur_logp && M.D)
        for (int c = 0; c < M.D; ++c)
          dur_logp[(size_t)b * M.D + c] = lg[(size_t)b * M.NOUT + M.V1p + c] - lse[s.Bp + b];
    }
    return RNNTG_OK;
  };
  st = run();
  mem.release();
  return st;
}

rnntg_status rnntg_step_prediction(rnntg_model* m, int batch, const int32_t* labels,
                                   const float* state, float* state_out) {
  if (!m) return fail(RNNTG_E_STATE, "model is null");
  if (m->dm.cell == RNNTG_CELL_SCRIPTED) return fail(RNNTG_E_VALUE, "not available for a scripted model");
  if (batch < 1 || batch > RB * MAXRB) return fail(RNNTG_E_VALUE, "bad batch");
  if (!labels || !state || !state_out) return fail(RNNTG_E_DIMENSION, "null buffer");
  const DevModel& M = m->dm;
  for (int b = 0; b < batch; ++b)
    if (labels[b] < 0 || labels[b] >= M.V1)  // embedding_lookup_into, tensor.cpp:499-502
      return fail(RNNTG_E_INDEX, "embedding id " + std::to_string(labels[b]) + " out of range");
  CK(cudaSetDevice(m->device));
  DevBuf mem;
  DevState s;
  rnntg_status st = alloc_state(m, mem, s, RNNTG_ALGO_FRAME_SYNC, batch, 1, 1, false);
  if (st) {
    mem.release();
    return st;
  }
  const bool lstm = M.cell == RNNTG_CELL_LSTM;
  const int W = lstm ? 2 * M.L * M.H : M.H;
  auto run = [&]() -> rnntg_status {
    for (int l = 0; l < M.L; ++l) {
      const int ho = lstm ? 2 * l * M.H : 0;
      CK(cudaMemcpy2D(s.h[l][0], sizeof(float) * M.Hp, state + ho, sizeof(float) * W,
                      sizeof(float) * M.H, batch, cudaMemcpyHostToDevice));
      if (lstm)
        CK(cudaMemcpy2D(s.c[l][0], sizeof(float) * M.Hp, state + ho + M.H, sizeof(float) * W,
                        sizeof(float) * M.H, batch, cudaMemcpyHostToDevice));
    }
    std::vector<int> ones(batch, 1);
    CK(cudaMemcpy(s.accept, ones.data(), sizeof(int) * batch, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s.last_label, labels, sizeof(int) * batch, cudaMemcpyHostToDevice));
    CK(cudaMemset(s.ctrl, 0, sizeof(Ctrl)));
    s.use_cond = 0;
    for (int l = 0; l < M.L; ++l) {
      if (lstm)
        pred_layer_kernel<1><<<dim3(M.GH / CT, s.nrb), NT, layer_smem(M, l)>>>(M, s, l);
      else
        pred_layer_kernel<0><<<dim3(M.GH / CT, s.nrb), NT, layer_smem(M, l)>>>(M, s, l);
      CK(cudaGetLastError());
    }
    CK(cudaDeviceSynchronize());
    for (int l = 0; l < M.L; ++l) {
      const int ho = lstm ? 2 * l * M.H : 0;
      CK(cudaMemcpy2D(state_out + ho, sizeof(float) * W, s.h[l][1], sizeof(float) * M.Hp,
                      sizeof(float) * M.H, batch, cudaMemcpyDeviceToHost));
      if (lstm)
        CK(cudaMemcpy2D(state_out + ho + M.H, sizeof(float) * W, s.c[l][1], sizeof(float) * M.Hp,
                        sizeof(float) * M.H, batch, cudaMemcpyDeviceToHost));
    }
    return RNNTG_OK;
  };
  st = run();
  mem.release();
  return st;
}

rnntg_status rnntg_time_kernel(rnntg_decoder* d, int which, int reps, float* avg_ms) {
  if (!d || !avg_ms || reps < 1) return fail(RNNTG_E_VALUE, "bad arguments");
  if (d->m->dm.cell == RNNTG_CELL_SCRIPTED) return fail(RNNTG_E_VALUE, "not available for a scripted model");
  if (!d->subs.empty()) return rnntg_time_kernel(d->subs[0], which, reps, avg_ms);
  CK(cudaSetDevice(d->m->device));
  const DevModel& M = d->m->dm;
  DevState s = d->st;
  s.use_cond = 0;
  s.max_iters = (long long)1 << 60;
  cudaStream_t st = d->stream;
  auto launch_one = [&]() -> cudaError_t {
    if (which == 0) return encproj_launch(d->enc, st);
    if (which == 10) {  // the persistent decode kernel alone (fp already projected)
      if (d->exec == RNNTG_EXEC_TENSOR) return launch_tc(d, st);
      if (d->exec != RNNTG_EXEC_PERSISTENT) return cudaErrorInvalidValue;
      void* args[1] = {&d->pp};
      return cudaLaunchCooperativeKernel((const void*)pk::persistent_kernel, dim3(d->pp.G),
                                         dim3(pk::NTH), args, d->psmem, st);
    }
    if (which >= 1 && which <= M.L) {
      const int l = which - 1;
      if (M.cell == RNNTG_CELL_LSTM)
        pred_layer_kernel<1><<<dim3(M.GH / CT, s.nrb), NT, layer_smem(M, l), st>>>(M, s, l);
      else
        pred_layer_kernel<0><<<dim3(M.GH / CT, s.nrb), NT, layer_smem(M, l), st>>>(M, s, l);
      return cudaGetLastError();
    }
    if (which == 8) {
      pred_proj_kernel<<<dim3(M.Jp / CT, s.nrb), NT, pp_smem(M), st>>>(M, s);
      return cudaGetLastError();
    }
    if (which == 9) {
      timing_prep_kernel<<<1, 256, 0, st>>>(s);
      joint_kernel<<<dim3(M.NCHT, s.nrb), NT, joint_smem(M), st>>>(M, s);
      return cudaGetLastError();
    }
    return cudaErrorInvalidValue;
  };
  timing_prep_kernel<<<1, 256, 0, st>>>(s);
  CK(cudaGetLastError());
  CK(launch_one());  // warm
  CK(cudaStreamSynchronize(st));
  float total = 0.0f;
  for (int r = 0; r < reps; ++r) {
    if (which == 9) {
      timing_prep_kernel<<<1, 256, 0, st>>>(s);
      CK(cudaGetLastError());
    }
    CK(cudaEventRecord(d->ev0, st));
    if (which == 9) {
      joint_kernel<<<dim3(M.NCHT, s.nrb), NT, joint_smem(M), st>>>(M, s);
      CK(cudaGetLastError());
    } else {
      CK(launch_one());
    }
    CK(cudaEventRecord(d->ev1, st));
    CK(cudaEventSynchronize(d->ev1));
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, d->ev0, d->ev1));
    total += ms;
  }
  *avg_ms = total / reps;
  d->launched = false;
  return RNNTG_OK;
}

rnntg_status rnntg_debug_trace(rnntg_decoder* d, unsigned long long* out, int n) {
  if (!d || !out) return fail(RNNTG_E_VALUE, "bad arguments");
  if (!d->subs.empty()) return rnntg_debug_trace(d->subs[0], out, n);  // first sub-batch
  CK(cudaStreamSynchronize(d->stream));
  if (d->tp.stamps) {  // RNNTG_STAMPS=1 (STAMPS builds): [64 step slots][G][16] globaltimer stamps
    const int tot = 64 * d->tp.G * 16;
    CK(cudaMemcpy(out, d->tp.stamps, sizeof(unsigned long long) * std::min(n, tot), cudaMemcpyDeviceToHost));
    return RNNTG_OK;
  }
  if (d->exec != RNNTG_EXEC_TENSOR || !d->tp.prof)
    return fail(RNNTG_E_STATE, "tracing needs the tensor executor and RNNTG_PROF=1");
  const int tot = (2 * ptc::NEV + d->tp.G) * ptc::PROF_WIN;
  CK(cudaMemcpy(out, d->tp.prof, sizeof(unsigned long long) * std::min(n, tot), cudaMemcpyDeviceToHost));
  return RNNTG_OK;
}

rnntg_status rnntg_debug_logits(rnntg_decoder* d, int step, float* out) {
  if (!d || !out || step < 0) return fail(RNNTG_E_VALUE, "bad arguments");
  if (d->exec != RNNTG_EXEC_TENSOR || !d->subs.empty())
    return fail(RNNTG_E_STATE, "logit dumps need the tensor executor (batch <= 256)");
  if (!d->bound) return fail(RNNTG_E_STATE, "captured decoder is not initialized (no inputs bound)");
  CK(cudaSetDevice(d->m->device));
  const size_t n = (size_t)d->B * (d->tp.V1 + d->tp.D);
  float* buf = nullptr;
  CK(cudaMalloc(&buf, n * sizeof(float)));
  cudaError_t e = cudaMemsetAsync(buf, 0, n * sizeof(float), d->stream);
  d->tp.dbg_logits = buf;
  d->tp.dbg_step = step;
  if (e == cudaSuccess) e = issue_persistent(d, d->stream);  // direct launch: the captured one has no dump
  d->tp.dbg_logits = nullptr;
  if (e == cudaSuccess) e = cudaStreamSynchronize(d->stream);
  if (e == cudaSuccess) e = cudaMemcpy(out, buf, n * sizeof(float), cudaMemcpyDeviceToHost);
  cudaFree(buf);
  if (e != cudaSuccess) return fail(RNNTG_E_CUDA, std::string("debug logits: ") + cudaGetErrorString(e));
  return RNNTG_OK;
}

rnntg_status rnntg_debug_profile(rnntg_decoder* d, unsigned long long* out16) {
  if (!d || !out16) return fail(RNNTG_E_VALUE, "bad arguments");
  if (d->exec != RNNTG_EXEC_PERSISTENT || !d->pp.prof)
    return fail(RNNTG_E_STATE, "profiling needs the persistent executor and RNNTG_PROF=1");
  CK(cudaStreamSynchronize(d->stream));
  CK(cudaMemcpy(out16, d->pp.prof, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  CK(cudaMemset(d->pp.prof, 0, 16 * sizeof(unsigned long long)));
  return RNNTG_OK;
}

rnntg_status rnntg_enc_proj(rnntg_model* m, int rows, const float* x, float* fp) {
  if (!m) return fail(RNNTG_E_STATE, "model is null");
  if (m->dm.cell == RNNTG_CELL_SCRIPTED) return fail(RNNTG_E_VALUE, "not available for a scripted model");
  if (rows < 1 || !x || !fp) return fail(RNNTG_E_DIMENSION, "bad arguments");
  CK(cudaSetDevice(m->device));
  const DevModel& M = m->dm;
  DevBuf mem;
  float *xd = nullptr, *od = nullptr;
  auto run = [&]() -> rnntg_status {
    CK(mem.alloc(&xd, (size_t)rows * M.Fp));
    CK(mem.alloc(&od, (size_t)rows * M.Jp));
    CK(cudaMemcpy2D(xd, sizeof(float) * M.Fp, x, sizeof(float) * M.F, sizeof(float) * M.F, rows,
                    cudaMemcpyHostToDevice));
    EncPlan plan;
    if (!encproj_plan(plan, M, xd, od, rows)) return fail(RNNTG_E_CUDA, "tensor map encode failed");
    CK(encproj_launch(plan, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy2D(fp, sizeof(float) * M.J, od, sizeof(float) * M.Jp, sizeof(float) * M.J, rows,
                    cudaMemcpyDeviceToHost));
    return RNNTG_OK;
  };
  rnntg_status st = run();
  mem.release();
  return st;
}

}  // extern "C"

namespace {
cudaError_t add_encproj(Builder& b, rnntg_decoder* d) {
  const DevModel& M = d->m->dm;
  const int rows = d->B * d->T;
  (void)M;
  (void)rows;
  return encproj_add_node(b.g, &b.last, &b.last_kernel, d->enc);
}
}  // namespace
