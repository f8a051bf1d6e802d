// mpm_api.cu -- C ABI + runtime of the B200-native differentiable MLS-MPM step.
// Declared in include/mpm.h.  Owns device memory, the tape (the paper's memo),
// the per-step launch schedule, the device error latch and per-kernel profiling.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl is resolved at run time (see nccl_api)

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/mpm.h"
#include "mpm_kernels.cuh"

using namespace mpm;

namespace {

enum KernelId {
  KI_SCAN, KI_SCATTER, KI_P2G, KI_G2P, KI_ZERO, KI_G2PT, KI_GRIDT, KI_P2GT, KI_MISC,
  KI_BANDP, KI_BANDU, KI_CTRL, KI_CTRLT, KI_FUSE, KI_MIG, KI_COUNT
};
const char* kKernelNames[KI_COUNT] = {"scan",  "scatter", "p2g",       "g2p",         "zero_adj", "g2p_T", "grid_T",
                                      "p2g_T", "misc",    "band_pack", "band_unpack", "ctrl",     "ctrl_T",
                                      "g2p2g", "migrate"};

struct PendingEvent {
  cudaEvent_t a, b;
  int kid;
};

// NCCL entry points, resolved on first use (slab mode only).  No link-time dependency: a
// process that loads libmpm before torch must not bind libnccl.so.2 to a different copy than
// the one torch needs; an already-loaded libnccl (torch's) is preferred.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};

const NcclApi* nccl_api() {
  // function-local static: initialised once, thread-safe (C++11)
  static const NcclApi* const api = []() -> const NcclApi* {
    static NcclApi a{};
    // an NCCL already in the process (e.g. torch's) first; else MPM_NCCL_LIB (the Python binding
    // points it at the NCCL torch bundles, so that a later `import torch` finds the NCCL it
    // was built against under the shared soname); else the loader's search path
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h)
      if (const char* p = getenv("MPM_NCCL_LIB"); p && *p) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    bool ok = h != nullptr;
#define NCCL_SYM(f)                                                  \
  if (ok) {                                                          \
    *reinterpret_cast<void**>(&a.f) = dlsym(h, "nccl" #f);            \
    ok = a.f != nullptr;                                             \
  }
    NCCL_SYM(GetUniqueId) NCCL_SYM(CommInitRank) NCCL_SYM(CommDestroy) NCCL_SYM(Send) NCCL_SYM(Recv)
    NCCL_SYM(AllReduce) NCCL_SYM(GroupStart) NCCL_SYM(GroupEnd) NCCL_SYM(GetErrorString)
#undef NCCL_SYM
    return ok ? &a : nullptr;
  }();
  return api;
}

}  // namespace

struct mpm_ctx_s {
  mpm_config cfg{};
  KParams P{};
  int D = 3, S = 24;
  cudaStream_t stream = nullptr;
  int n_sm = 148;
  int occ_scatter = 2, occ_scatter_adj = 2, occ_g2p = 2, occ_p2gT = 2;
  int tape_len = 0;
  // NEXT N2 checkpointing: the tape holds steps [seg0, seg0 + tape_cap] (segment-local slots);
  // with checkpoint_every = k > 0, full states are checkpointed every k steps and the
  // backward recomputes each earlier segment from its checkpoint
  int tape_cap = 0, seg0 = 0, seg_end = 0, ck = 0, n_ck = 0, ck_valid = 0;
  int res_end = 0;  // the states of steps [seg0, res_end] on the tape are valid
  int fused_grid = -1;  // fused forward: the step whose grid the previous G2P2G already built
  int occ_fuse = 2;
  float* ck_state = nullptr;
  int* ck_orig = nullptr;
  bool has_state = false, has_act = false, has_grad = false, poisoned = false;
  std::string last_error;
  int64_t launches = 0;
  MigParams M{0, INT32_MIN, INT32_MAX, 0};  // migrating slab mode
  int latch_step = -1;  // step of the last latched device error (check_latch)
  // tape
  float* tape_state = nullptr;
  int* tape_perm = nullptr;
  int* tape_orig = nullptr;
  int* tape_bs = nullptr;
  int* tape_slot = nullptr;
  int4* tape_occ = nullptr;  // per step: occupied-block work items {block, first, count, 0}
  int* tape_touch = nullptr;
  int* info = nullptr;
  float4* arena = nullptr;
  size_t arena_slots = 0;
  // work buffers
  int* key = nullptr;
  int* cnt = nullptr;
  int2* tmp_pk = nullptr;
  int* scratch = nullptr;
  int* hist2 = nullptr;
  int3* tile_sums = nullptr;
  ScanTileState scan{};   // single-pass binning scan: tile flags / aggregates / prefixes / ticket
  unsigned scan_epoch = 0;
  int n_tiles = 0;
  ErrLatch* err = nullptr;
  int* dbad = nullptr;
  float4* prm = nullptr;
  int* aid = nullptr;
  float* E = nullptr;
  float* nu = nullptr;
  float* act = nullptr;
  float* gA = nullptr;
  float* gB = nullptr;
  float4* agrid = nullptr;
  float4* agrid1 = nullptr;
  unsigned* bflag = nullptr;
  float* dmu = nullptr;
  float* dlam = nullptr;
  float* dmass = nullptr;
  std::map<int, float*> seeds;  // per-step additive seeds (user-order AoS x|v|F|C), N4
  float* da = nullptr;
  float* stage = nullptr;
  std::vector<void*> allocs;
  // slab mode: x-slab [x_lo, x_hi), boundary windows of 2*halo block-planes
  bool slab = false, left = false, right = false;
  int x_lo = 0, x_hi = 0, halo = 0;
  int band_blocks = 0, gb_lo = 0, gb_hi = 0;  // blocks per window, first block of each window
  float4 *send_lo = nullptr, *send_hi = nullptr, *recv_lo = nullptr, *recv_hi = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  // migrating slab mode (mpm_set_slab_migrating): ownership by base_x at every step; user arrays
  // span the whole body (NU particles), storage holds up to P.NT (the capacity)
  bool mig = false;
  size_t NU = 0;                 // user-array length (= P.NT outside migrating mode)
  size_t mig_floats = 0;         // floats per migrant buffer (header + mig_cap records)
  float* mig_send_tape = nullptr;  // [tape_cap][2][mig_floats]: leavers of step t (kept for the backward)
  float* mig_recv_tape = nullptr;  // [tape_cap][2][mig_floats]: arrivals of step t
  float *rev_send[2] = {nullptr, nullptr}, *rev_recv[2] = {nullptr, nullptr};  // [mig_cap][S] adjoints
  int* members = nullptr;        // set_state: this slab's user indices (storage order 0)
  // host-staged transport (mpm_set_transport): the exchanges go through a caller callback
  mpm_transport_fn transport = nullptr;
  void* transport_user = nullptr;
  float* host_stage = nullptr;   // pinned: send_l | send_r | recv_l | recv_r
  size_t host_stage_floats = 0;
  // NEXT N1 controller: a_t = tanh(W z_t + b)
  bool ctrl = false, ctrl_grad_valid = false;
  float *ctrl_W = nullptr, *ctrl_b = nullptr, *ctrl_target = nullptr, *ctrl_Minv = nullptr, *ctrl_acc = nullptr;
  int* ctrl_cnt = nullptr;
  float *ctrl_M = nullptr, *ztape = nullptr, *gpre_tape = nullptr, *ctrl_gz = nullptr;
  int* ctrl_n = nullptr;
  float *ctrl_gW = nullptr, *ctrl_gb = nullptr, *ctrl_gt = nullptr;
  float* bcur = nullptr;  // backward: adjoint of the current step (storage order)
  float* bnxt = nullptr;
  // profiling
  bool profiling = false;
  // mpm_set_graphs: step loops captured once per (direction, start, length) and replayed as
  // CUDA graphs; the host-side effects of a capture (launch count, scan epochs) are replayed too
  bool graphs = false;
  struct GraphRec {
    int dir, t0, n;
    cudaGraphExec_t exec;
    int64_t launches;
    unsigned epochs;
  };
  std::vector<GraphRec> gcache;
  bool pdl = true;  // programmatic dependent launches on the step path (MPM_PDL=0 disables)
  bool split = false;  // small problem: the gathers split blocks into particle ranges
  bool mass_grad = false;  // N3: compute dL/dm_p in P2G^T (opt-in)
  bool mass_grad_valid = false;
  std::vector<PendingEvent> pending;
  std::vector<cudaEvent_t> event_pool;
  double prof_ms[KI_COUNT] = {};
  int64_t prof_n[KI_COUNT] = {};
};

namespace {

// the reason the calling thread's last mpm_create failed (read by mpm_last_error(NULL))
thread_local std::string g_create_error;

mpm_status fail(mpm_ctx c, mpm_status s, const std::string& msg) {
  if (c) c->last_error = msg;
  return s;
}

mpm_status cuda_fail(mpm_ctx c, cudaError_t e, const char* where) {
  return fail(c, MPM_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                                   \
  do {                                                             \
    cudaError_t e_ = (call);                                       \
    if (e_ != cudaSuccess) return cuda_fail(c, e_, #call);         \
  } while (0)

template <class T>
mpm_status dalloc(mpm_ctx c, T** p, size_t count) {
  void* q = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(&q, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, MPM_ERR_OOM, "cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed");
  }
  c->allocs.push_back(q);
  *p = static_cast<T*>(q);
  return MPM_OK;
}

cudaEvent_t get_event(mpm_ctx c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Launch wrapper: counts launches and (when profiling) brackets the kernel with events.
template <class F>
void launch(mpm_ctx c, int kid, F&& f) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->profiling) {
    a = get_event(c);
    b = get_event(c);
    cudaEventRecord(a, c->stream);
  }
  f();
  ++c->launches;
  if (c->profiling) {
    cudaEventRecord(b, c->stream);
    c->pending.push_back({a, b, kid});
  }
}

void drain_profile(mpm_ctx c) {
  for (auto& p : c->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      c->prof_ms[p.kid] += ms;
      c->prof_n[p.kid] += 1;
    }
    c->event_pool.push_back(p.a);
    c->event_pool.push_back(p.b);
  }
  c->pending.clear();
}

// Launch of a step-path kernel: with c->pdl, as a programmatic dependent launch (the
// kernel begins with MPM_PDL_ENTRY, so it still observes every write of its predecessor).
template <class... KA, class... A>
void kx(mpm_ctx c, void (*k)(KA...), dim3 g, dim3 b, size_t smem, A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = c->pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

size_t NTs(mpm_ctx c) { return (size_t)c->P.NT; }

void drop_graphs(mpm_ctx c) {
  if (c->gcache.empty()) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& g : c->gcache) cudaGraphExecDestroy(g.exec);
  c->gcache.clear();
}

// tape slot of global step t (segment-local; the caller guarantees seg0 <= t <= seg0 + tape_cap)
size_t ti(mpm_ctx c, int t) { return (size_t)(t - c->seg0); }
size_t recf(mpm_ctx c) { return rec_floats(c->S, NTs(c)); }  // floats of one particle-record buffer
float* state_at(mpm_ctx c, int t) { return c->tape_state + ti(c, t) * recf(c); }
int* perm_at(mpm_ctx c, int t) { return c->tape_perm + ti(c, t) * NTs(c); }
int* orig_at(mpm_ctx c, int t) { return c->tape_orig + ti(c, t) * NTs(c); }
int* bs_at(mpm_ctx c, int t) { return c->tape_bs + ti(c, t) * (c->P.NBT + 1); }
int* slot_at(mpm_ctx c, int t) { return c->tape_slot + ti(c, t) * c->P.NBT; }
int4* occ_at(mpm_ctx c, int t) { return c->tape_occ + ti(c, t) * c->P.NBT; }
int* touch_at(mpm_ctx c, int t) { return c->tape_touch + ti(c, t) * c->P.NBT; }
int* info_at(mpm_ctx c, int t) { return c->info + ti(c, t) * kInfo; }
// migrating slab mode: buffers of step t
float* mig_send_at(mpm_ctx c, int t, int side) { return c->mig_send_tape + ((size_t)ti(c, t) * 2 + side) * c->mig_floats; }
float* mig_recv_at(mpm_ctx c, int t, int side) { return c->mig_recv_tape + ((size_t)ti(c, t) * 2 + side) * c->mig_floats; }
const int* nslot_at(mpm_ctx c, int t) { return c->mig ? info_at(c, t) + I_NSLOT : nullptr; }
size_t rev_floats(mpm_ctx c) { return (size_t)c->M.mig_cap * c->S; }

bool on_tape(mpm_ctx c, int t) { return t >= c->seg0 && t <= c->res_end && t <= c->tape_len; }
float* ck_state_of(mpm_ctx c, int i) { return c->ck_state + (size_t)i * recf(c); }
int* ck_orig_of(mpm_ctx c, int i) { return c->ck_orig + (size_t)i * NTs(c); }

int grid1d(size_t n, int bs = 256) { return (int)((n + bs - 1) / bs); }

// Read the device error latch (after a stream sync) and turn it into a status.
mpm_status check_latch(mpm_ctx c) {
  ErrLatch h{};
  cudaError_t e = cudaMemcpy(&h, c->err, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(c, e, "error latch readback");
  if (h.code == 0) return MPM_OK;
  c->latch_step = h.step;
  char buf[256];
  if (h.code == E_DOMAIN) {
    snprintf(buf, sizeof buf, "particle %d left the domain (base index outside [0, res-3]) at step %d", h.particle, h.step);
    c->poisoned = true;
    return fail(c, MPM_ERR_OUT_OF_DOMAIN, buf);
  }
  if (h.code == E_INVERTED) {
    snprintf(buf, sizeof buf, "inverted element: det F <= 0 for particle %d at step %d", h.particle, h.step);
    c->poisoned = true;
    return fail(c, MPM_ERR_INVERTED, buf);
  }
  if (h.code == E_TAPE_FULL) {
    snprintf(buf, sizeof buf, "grid-slot arena full at step %d (%d touched blocks); raise config.grid_slots",
             h.step, h.particle);
    c->poisoned = true;
    return fail(c, MPM_ERR_TAPE_FULL, buf);
  }
  if (h.code == E_FUSE) {
    snprintf(buf, sizeof buf, "particle %d moved more than the fused step's grid dilation allows at step %d "
             "(fuse_g2p2g needs |v| dt < dx)", h.particle, h.step);
    c->poisoned = true;
    return fail(c, MPM_ERR_CFL, buf);
  }
  if (h.code == E_SLAB) {
    snprintf(buf, sizeof buf, "particle %d left its slab's halo (base x outside [%d, %d]) at step %d", h.particle,
             c->P.slab_lo, c->P.slab_hi, h.step);
    c->poisoned = true;
    return fail(c, MPM_ERR_OUT_OF_SLAB, buf);
  }
  if (h.code == E_MIGRATE) {
    snprintf(buf, sizeof buf, "migrating slab mode at step %d: more leavers per side than mig_cap (%d), more "
             "particles than the storage capacity, or a particle that crossed a whole slab (%d)", h.step,
             c->M.mig_cap, h.particle);
    c->poisoned = true;
    return fail(c, MPM_ERR_MIGRATE, buf);
  }
  snprintf(buf, sizeof buf, "device error code %d", h.code);
  return fail(c, MPM_ERR_CUDA, buf);
}

mpm_status sync_and_check(mpm_ctx c, const char* where) {
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (c->profiling) drain_profile(c);
  if (e != cudaSuccess) return cuda_fail(c, e, where);
  return check_latch(c);
}

template <int D>
void launch_keys(mpm_ctx c, int t) {
  const KParams& P = c->P;
  // storage order 0 = user order (identity orig) outside migrating mode; there set_state wrote
  // the members' user indices
  int* orig0 = (t == 0 && !c->mig) ? orig_at(c, 0) : nullptr;
  launch(c, KI_MISC, [&] {
    k_init_keys<D><<<grid1d(P.NT), 256, 0, c->stream>>>(P, state_at(c, t), c->key, c->cnt, orig0, c->err,
                                                         nslot_at(c, t), c->M);
  });
}

// Fill StepArgs for step t.
StepArgs step_args(mpm_ctx c, int t) {
  StepArgs A{};
  A.st = state_at(c, t);
  A.perm = perm_at(c, t);
  A.tmp_pk = c->tmp_pk;
  A.key = c->key;
  A.scratch = c->scratch;
  A.orig = orig_at(c, t);
  A.prm = c->prm;
  A.aid = c->aid;
  A.act = c->act;
  A.block_start = bs_at(c, t);
  A.occ_list = occ_at(c, t);
  A.slot_of = slot_at(c, t);
  A.touched_list = touch_at(c, t);
  A.info_t = info_at(c, t);
  A.grid = c->arena;
  A.tgrid = c->arena;
  A.st_next = state_at(c, t + 1);
  A.orig_next = orig_at(c, t + 1);
  A.key_next = c->key;
  A.cnt = c->cnt;
  A.dmu = c->dmu;
  A.dlam = c->dlam;
  A.dmass = c->dmass;
  A.da = c->da;
  A.err = c->err;
  A.t = t;
  return A;
}

void launch_scatter(mpm_ctx c, int t, const int* za, const int* zb);

// binning tables of step t from the keys/histogram of state t
template <int D>
void launch_bin(mpm_ctx c, int t) {
  const KParams& P = c->P;
  const unsigned epoch = (++c->scan_epoch) & 0x3fffffffu;
  launch(c, KI_SCAN, [&] {
    kx(c, k_scan_lookback<D>, dim3(c->n_tiles), dim3(kScanTile), 0, P, c->cnt, c->scan, epoch, c->n_tiles,
       info_at(c, t), bs_at(c, t), occ_at(c, t), info_at(c, t), ti(c, t) ? info_at(c, t - 1) : nullptr,
       slot_at(c, t), touch_at(c, t), c->err, t);
  });
  launch_scatter(c, t, info_at(c, t), nullptr);
}

// block-grouping of step t's particles; zeroes the grid slots of the step records za, zb
void launch_scatter(mpm_ctx c, int t, const int* za, const int* zb) {
  const KParams& P = c->P;
  launch(c, KI_SCATTER, [&] {
    kx(c, k_scatter, dim3(std::max(1, std::min(grid1d(P.NT), c->n_sm * MPM_SCAT_CTAS))), dim3(256), 0, P.NT, c->key, bs_at(c, t),
       c->cnt, c->tmp_pk, za, zb, c->arena, nslot_at(c, t));
  });
}

// NEXT N2 fused forward: binning of step t (info_bin non-null) and/or the dilated grid-slot
// table of step t+1 (grid = true)
template <int D>
void launch_bin_fused(mpm_ctx c, int t, bool bin, bool grid) {
  const KParams& P = c->P;
  const unsigned epoch = (++c->scan_epoch) & 0x3fffffffu;
  launch(c, KI_SCAN, [&] {
    kx(c, k_scan_lookback<D, true>, dim3(c->n_tiles), dim3(kScanTile), 0, P, c->cnt, c->scan, epoch, c->n_tiles,
       bin ? info_at(c, t) : nullptr, bs_at(c, t), occ_at(c, t), grid ? info_at(c, t + 1) : nullptr, info_at(c, t),
       grid ? slot_at(c, t + 1) : nullptr, grid ? touch_at(c, t + 1) : nullptr, c->err, t);
  });
}

bool has_nbr(mpm_ctx c) { return c->slab && (c->left || c->right); }

// slab mode: boundary windows of step t's grid -> send buffers (forward: tape arena; adjoint:
// the step's adjoint buffer)
void launch_band_pack(mpm_ctx c, int t, bool adj, const float4* g) {
  launch(c, KI_BANDP, [&] {
    kx(c, k_band_pack, dim3(c->n_sm * 4), dim3(256), 0, c->band_blocks, c->gb_lo, c->gb_hi, slot_at(c, t), info_at(c, t),
                                                    adj, g, c->left ? c->send_lo : nullptr,
                                                    c->right ? c->send_hi : nullptr);
  });
}
void launch_band_unpack(mpm_ctx c, int t, bool adj, float4* g) {
  launch(c, KI_BANDU, [&] {
    kx(c, k_band_unpack, dim3(c->n_sm * 4), dim3(256), 0, c->band_blocks, c->gb_lo, c->gb_hi, slot_at(c, t), info_at(c, t),
                                                      adj, g, c->left ? c->recv_lo : nullptr,
                                                      c->right ? c->recv_hi : nullptr);
  });
}
size_t band_floats(mpm_ctx c) { return (size_t)c->band_blocks * kCPB * 4; }

// Exchange with the x-neighbours (ranks ordered by slab): send_l -> left, send_r -> right,
// recv_l <- left, recv_r <- right, n floats each (sides without a neighbour are skipped).
// NCCL: grouped send/recv on the library stream.  With a transport callback (mpm_set_transport):
// the stream is synchronised, the send buffers staged in pinned host memory, the callback does
// the exchange, and the receive buffers are copied back -- no kernel waits on another rank.
mpm_status exchange_pair(mpm_ctx c, int kind, const float* send_l, const float* send_r, float* recv_l, float* recv_r,
                         size_t n) {
  if (c->transport) {
    if (c->host_stage_floats < 4 * n) {
      if (c->host_stage) cudaFreeHost(c->host_stage);
      c->host_stage = nullptr;
      c->host_stage_floats = 0;
      CK(cudaMallocHost(&c->host_stage, 4 * n * sizeof(float)));
      c->host_stage_floats = 4 * n;
    }
    float* h = c->host_stage;
    if (c->left) CK(cudaMemcpyAsync(h, send_l, n * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    if (c->right) CK(cudaMemcpyAsync(h + n, send_r, n * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const int rc = c->transport(c->transport_user, kind, c->left ? h : nullptr, c->right ? h + n : nullptr,
                                c->left ? h + 2 * n : nullptr, c->right ? h + 3 * n : nullptr, n * sizeof(float));
    if (rc != 0) return fail(c, MPM_ERR_COMM, "transport callback failed (" + std::to_string(rc) + ")");
    if (c->left) CK(cudaMemcpyAsync(recv_l, h + 2 * n, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    if (c->right) CK(cudaMemcpyAsync(recv_r, h + 3 * n, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    return MPM_OK;
  }
  const NcclApi* N = nccl_api();  // non-null: the communicator exists
  ncclResult_t r = N->GroupStart();
  if (r == ncclSuccess && c->left) r = N->Send(send_l, n, ncclFloat, c->rank - 1, c->comm, c->stream);
  if (r == ncclSuccess && c->left) r = N->Recv(recv_l, n, ncclFloat, c->rank - 1, c->comm, c->stream);
  if (r == ncclSuccess && c->right) r = N->Send(send_r, n, ncclFloat, c->rank + 1, c->comm, c->stream);
  if (r == ncclSuccess && c->right) r = N->Recv(recv_r, n, ncclFloat, c->rank + 1, c->comm, c->stream);
  ncclResult_t r2 = N->GroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) return fail(c, MPM_ERR_COMM, std::string("slab exchange: ") + N->GetErrorString(r));
  return MPM_OK;
}

// the grid windows (forward after P2G, backward after G2P^T)
mpm_status exchange_nccl(mpm_ctx c) {
  return exchange_pair(c, MPM_XCHG_WINDOW, (const float*)c->send_lo, (const float*)c->send_hi, (float*)c->recv_lo,
                       (float*)c->recv_hi, band_floats(c));
}

// in-place sum over the slab ranks of n floats (NCCL all-reduce, or the transport's REDUCE)
mpm_status allreduce_sum(mpm_ctx c, float* d, size_t n) {
  if (n == 0) return MPM_OK;
  if (c->transport) {
    if (c->host_stage_floats < n) {
      if (c->host_stage) cudaFreeHost(c->host_stage);
      c->host_stage = nullptr;
      c->host_stage_floats = 0;
      CK(cudaMallocHost(&c->host_stage, n * sizeof(float)));
      c->host_stage_floats = n;
    }
    CK(cudaMemcpyAsync(c->host_stage, d, n * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const int rc = c->transport(c->transport_user, MPM_XCHG_REDUCE, c->host_stage, nullptr, nullptr, nullptr,
                                n * sizeof(float));
    if (rc != 0) return fail(c, MPM_ERR_COMM, "transport callback failed (" + std::to_string(rc) + ")");
    CK(cudaMemcpyAsync(d, c->host_stage, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    return MPM_OK;
  }
  const NcclApi* N = nccl_api();
  ncclResult_t r = N->AllReduce(d, d, n, ncclFloat, ncclSum, c->comm, c->stream);
  if (r != ncclSuccess) return fail(c, MPM_ERR_COMM, std::string("all-reduce: ") + N->GetErrorString(r));
  return MPM_OK;
}

bool has_xchg(mpm_ctx c) { return c->comm != nullptr || c->transport != nullptr; }

// in-process transport (mpm_group_*): contexts in slab order on one stream
mpm_status exchange_local(mpm_ctx* cs, int n) {
  for (int i = 0; i + 1 < n; ++i) {
    mpm_ctx a = cs[i], b = cs[i + 1];
    mpm_ctx c = a;
    const size_t bytes = band_floats(a) * sizeof(float);
    CK(cudaMemcpyAsync(b->recv_lo, a->send_hi, bytes, cudaMemcpyDeviceToDevice, a->stream));
    CK(cudaMemcpyAsync(a->recv_hi, b->send_lo, bytes, cudaMemcpyDeviceToDevice, a->stream));
  }
  return MPM_OK;
}

// migrating slab mode, in process: the migrant records of step t (forward) ...
mpm_status exchange_local_mig(mpm_ctx* cs, int n, int t) {
  for (int i = 0; i + 1 < n; ++i) {
    mpm_ctx a = cs[i], b = cs[i + 1];
    mpm_ctx c = a;
    const size_t bytes = a->mig_floats * sizeof(float);
    CK(cudaMemcpyAsync(mig_recv_at(b, t, 0), mig_send_at(a, t, 1), bytes, cudaMemcpyDeviceToDevice, a->stream));
    CK(cudaMemcpyAsync(mig_recv_at(a, t, 1), mig_send_at(b, t, 0), bytes, cudaMemcpyDeviceToDevice, a->stream));
  }
  return MPM_OK;
}

// ... and the adjoints of the arrivals going back (backward)
mpm_status exchange_local_rev(mpm_ctx* cs, int n) {
  for (int i = 0; i + 1 < n; ++i) {
    mpm_ctx a = cs[i], b = cs[i + 1];
    mpm_ctx c = a;
    const size_t bytes = rev_floats(a) * sizeof(float);
    CK(cudaMemcpyAsync(b->rev_recv[0], a->rev_send[1], bytes, cudaMemcpyDeviceToDevice, a->stream));
    CK(cudaMemcpyAsync(a->rev_recv[1], b->rev_send[0], bytes, cudaMemcpyDeviceToDevice, a->stream));
  }
  return MPM_OK;
}

// forward step t = phase A (binning, P2G [, window pack]) | exchange | phase B ([unpack,] G2P)
// N2: the tape is full at step t (t - seg0 == tape_cap): state t becomes checkpoint t / k and
// the first slot of a new segment (its keys / histogram are already in the work buffers)
void roll_segment(mpm_ctx c, int t) {
  const size_t bs = recf(c) * sizeof(float), bo = NTs(c) * sizeof(int);
  const int i = t / c->ck;
  cudaMemcpyAsync(ck_state_of(c, i), state_at(c, t), bs, cudaMemcpyDeviceToDevice, c->stream);
  cudaMemcpyAsync(ck_orig_of(c, i), orig_at(c, t), bo, cudaMemcpyDeviceToDevice, c->stream);
  cudaMemcpyAsync(c->tape_state, state_at(c, t), bs, cudaMemcpyDeviceToDevice, c->stream);
  cudaMemcpyAsync(c->tape_orig, orig_at(c, t), bo, cudaMemcpyDeviceToDevice, c->stream);
  c->seg0 = t;
  c->res_end = t;
  c->ck_valid = std::max(c->ck_valid, i + 1);
}

template <int D>
void forward_phase_a(mpm_ctx c, int t) {
  const KParams& P = c->P;
  if (c->ck && t - c->seg0 == c->tape_cap) roll_segment(c, t);
  if (c->ctrl)  // N1: a_t = tanh(W z_t + b) from state t, before P2G reads act[t]
    launch(c, KI_CTRL, [&] {
      kx(c, k_ctrl_observe<D>, dim3(c->n_sm * 4), dim3(256), 0, P, state_at(c, t), orig_at(c, t), c->prm, c->aid,
                                                             c->ctrl_acc, c->ctrl_cnt, c->ctrl_W, c->ctrl_b,
                                                             c->ctrl_target, c->ctrl_Minv, c->act,
                                                             c->ztape + (size_t)t * P.B * P.nz, t);
    });
  launch_bin<D>(c, t);
  StepArgs A = step_args(c, t);
  const int nblk = std::max(1, std::min(P.NBT, c->n_sm * c->occ_scatter));
  if (P.material == 1)  // fixed-corotated (R21)
    launch(c, KI_P2G, [&] { kx(c, k_block_scatter<D, false, 1>, dim3(nblk), dim3(kThreads), scatter_dyn_smem<D, false>(), P, A); });
  else
    launch(c, KI_P2G, [&] { kx(c, k_block_scatter<D, false>, dim3(nblk), dim3(kThreads), scatter_dyn_smem<D, false>(), P, A); });
  if (has_nbr(c)) launch_band_pack(c, t, false, c->arena);
}

template <int D>
void forward_phase_b(mpm_ctx c, int t) {
  const KParams& P = c->P;
  c->res_end = t + 1;
  if (has_nbr(c)) launch_band_unpack(c, t, false, c->arena);
  StepArgs A = step_args(c, t);
  const int ng = std::max(1, std::min(P.NBT, c->n_sm * c->occ_g2p));
  launch(c, KI_G2P, [&] {
    if (c->split) kx(c, k_g2p<D, true>, dim3(ng), dim3(kThreads), 0, P, A);  // small problems: blocks split
    else kx(c, k_g2p<D>, dim3(ng), dim3(kThreads), 0, P, A);
  });
  if (c->mig) {  // migrating slab mode: the particles of state t+1 that left the slab
    for (int side = 0; side < 2; ++side) cudaMemsetAsync(mig_send_at(c, t, side), 0, Mig<D>::HDR * sizeof(float), c->stream);
    launch(c, KI_MIG, [&] {
      kx(c, k_mig_leavers<D>, dim3(c->n_sm * 4), dim3(256), 0, P, c->M, (const int*)bs_at(c, t), (const float*)state_at(c, t + 1),
         (const int*)orig_at(c, t + 1), c->key, c->cnt, mig_send_at(c, t, 0), mig_send_at(c, t, 1), c->err, t);
    });
  }
}

// migrating slab mode, after the migrant exchange of step t: append the arrivals to state t+1
template <int D>
void forward_phase_c(mpm_ctx c, int t) {
  const KParams& P = c->P;
  launch(c, KI_MIG, [&] {
    kx(c, k_mig_append<D>, dim3(c->n_sm), dim3(256), 0, P, c->M, c->left ? (const float*)mig_recv_at(c, t, 0) : nullptr,
       c->right ? (const float*)mig_recv_at(c, t, 1) : nullptr, (const int*)bs_at(c, t), state_at(c, t + 1),
       orig_at(c, t + 1), c->key, c->cnt, info_at(c, t + 1), c->err, t);
  });
}

// migrating slab mode, before G2P^T of step t: arrivals' adjoints out, leavers' adjoints in
template <int D>
void backward_mig_pack(mpm_ctx c, int t) {
  launch(c, KI_MIG, [&] {
    kx(c, k_mig_rev_pack<D>, dim3(c->n_sm), dim3(256), 0, c->P, c->M, c->left ? (const float*)mig_recv_at(c, t, 0) : nullptr,
       c->right ? (const float*)mig_recv_at(c, t, 1) : nullptr, (const int*)bs_at(c, t), (const float*)c->bcur,
       c->rev_send[0], c->rev_send[1]);
  });
}
template <int D>
void backward_mig_unpack(mpm_ctx c, int t) {
  launch(c, KI_MIG, [&] {
    kx(c, k_mig_rev_unpack<D>, dim3(c->n_sm), dim3(256), 0, c->P, c->M, c->left ? (const float*)mig_send_at(c, t, 0) : nullptr,
       c->right ? (const float*)mig_send_at(c, t, 1) : nullptr, (const float*)c->rev_recv[0],
       (const float*)c->rev_recv[1], c->bcur);
  });
}

// NEXT N2 fused forward (config.fuse_g2p2g): step t's G2P also scatters step t+1's P2G
// (k_g2p2g) when step t+1 is in the same forward range and segment; grid t+1's slot map is
// then the dilation of step t's occupied blocks.  Per fused step: scan (binning t + grid t+1
// table) -> k_scatter (block grouping, zero grid t+1) -> k_g2p2g (cell sort of t, G2P, P2G
// of t+1): 3 launches, one particle pass.  A step whose grid is not yet built (the first
// of a range or of a segment) runs the unfused P2G first.
// A slab with neighbours (Lagrangian ownership) sums its windows of grid t+1 between two
// G2P2G launches: grid t+1 is complete before the G2P of step t+1 reads it.  Not fused: the
// migrating slab mode (arrivals are appended to state t+1 after its G2P) and the controller.
bool fuse_on(mpm_ctx c) { return c->cfg.fuse_g2p2g && !c->ctrl && !c->mig; }

template <int D, bool SORT, bool SCAT>
void launch_fused(mpm_ctx c, const StepArgs& A) {
  const KParams& P = c->P;
  const size_t dyn = SCAT ? fuse_dyn_smem<D>() : 0;
  if (c->split) {  // small problems: blocks shared by several CTAs (work_parts)
    const int ng = std::max(1, std::min(8 * P.NBT, c->n_sm * c->occ_fuse));
    if (P.material == 1) kx(c, k_g2p2g<D, 1, SORT, SCAT, true>, dim3(ng), dim3(kThreads), dyn, P, A);
    else kx(c, k_g2p2g<D, 0, SORT, SCAT, true>, dim3(ng), dim3(kThreads), dyn, P, A);
    return;
  }
  const int ng = std::max(1, std::min(P.NBT, c->n_sm * c->occ_fuse));
  if (P.material == 1) kx(c, k_g2p2g<D, 1, SORT, SCAT>, dim3(ng), dim3(kThreads), dyn, P, A);
  else kx(c, k_g2p2g<D, 0, SORT, SCAT>, dim3(ng), dim3(kThreads), dyn, P, A);
}

// A fused step in two halves around the slab-window exchanges (a slab with neighbours sums its
// windows of grid t after the unfused P2G that starts a range, and of grid t+1 after each
// G2P2G).  Part a: start of a range or segment -- binning of t and the unfused P2G of step t
// (returns true: grid t was just built and, in slab mode, its windows are packed).
template <int D>
bool fused_part_a(mpm_ctx c, int t, int t_end) {
  const KParams& P = c->P;
  if (c->ck && t - c->seg0 == c->tape_cap) {
    roll_segment(c, t);
    c->fused_grid = -1;
  }
  if (c->fused_grid == t) return false;
  const bool next = t + 1 < t_end && (int)ti(c, t + 1) < c->tape_cap;
  StepArgs A = step_args(c, t);
  const unsigned epoch = (++c->scan_epoch) & 0x3fffffffu;
  launch(c, KI_SCAN, [&] {
    kx(c, k_scan_lookback<D>, dim3(c->n_tiles), dim3(kScanTile), 0, P, c->cnt, c->scan, epoch, c->n_tiles,
       info_at(c, t), bs_at(c, t), occ_at(c, t), info_at(c, t), ti(c, t) ? info_at(c, t - 1) : nullptr,
       slot_at(c, t), touch_at(c, t), c->err, t);
  });
  if (next) launch_bin_fused<D>(c, t, false, true);
  launch_scatter(c, t, info_at(c, t), next ? info_at(c, t + 1) : nullptr);
  const int nblk = std::max(1, std::min(P.NBT, c->n_sm * c->occ_scatter));
  launch(c, KI_P2G, [&] {
    if (P.material == 1) kx(c, k_block_scatter<D, false, 1>, dim3(nblk), dim3(kThreads), scatter_dyn_smem<D, false>(), P, A);
    else kx(c, k_block_scatter<D, false>, dim3(nblk), dim3(kThreads), scatter_dyn_smem<D, false>(), P, A);
  });
  if (has_nbr(c)) launch_band_pack(c, t, false, c->arena);
  return true;
}

// Part b: the G2P of step t, fused with step t+1's P2G when t+1 is in the range and segment
// (returns true: grid t+1 was built and, in slab mode, its windows are packed).
template <int D>
bool fused_part_b(mpm_ctx c, int t, int t_end, bool built) {
  const KParams& P = c->P;
  const bool next = t + 1 < t_end && (int)ti(c, t + 1) < c->tape_cap;
  StepArgs A = step_args(c, t);
  A.slot_next = next ? slot_at(c, t + 1) : nullptr;
  if (built) {
    if (has_nbr(c)) launch_band_unpack(c, t, false, c->arena);
    if (next) {
      launch(c, KI_FUSE, [&] { launch_fused<D, false, true>(c, A); });
    } else {
      const int ng = std::max(1, std::min(P.NBT, c->n_sm * c->occ_g2p));
      launch(c, KI_G2P, [&] {
        if (c->split) kx(c, k_g2p<D, true>, dim3(ng), dim3(kThreads), 0, P, A);
        else kx(c, k_g2p<D>, dim3(ng), dim3(kThreads), 0, P, A);
      });
    }
  } else {
    launch_bin_fused<D>(c, t, true, next);
    launch_scatter(c, t, next ? info_at(c, t + 1) : nullptr, nullptr);
    launch(c, KI_FUSE, [&] {
      if (next) launch_fused<D, true, true>(c, A);
      else launch_fused<D, true, false>(c, A);
    });
  }
  c->res_end = t + 1;
  c->fused_grid = next ? t + 1 : -1;
  if (next && has_nbr(c)) launch_band_pack(c, t + 1, false, c->arena);
  return next;
}

// forward steps [t0, t1) (slab mode: with the window exchange between the phases)
template <int D>
mpm_status forward_range(mpm_ctx c, int t0, int t1) {
  c->fused_grid = -1;
  if (fuse_on(c)) {
    for (int t = t0; t < t1; ++t) {
      const bool built = fused_part_a<D>(c, t, t1);
      if (built && has_nbr(c)) {
        mpm_status s = exchange_nccl(c);
        if (s) return s;
      }
      const bool next = fused_part_b<D>(c, t, t1, built);
      if (next && has_nbr(c)) {
        mpm_status s = exchange_nccl(c);
        if (s) return s;
        launch_band_unpack(c, t + 1, false, c->arena);
      }
    }
    return MPM_OK;
  }
  for (int t = t0; t < t1; ++t) {
    forward_phase_a<D>(c, t);
    if (has_nbr(c)) {
      mpm_status s = exchange_nccl(c);
      if (s) return s;
    }
    forward_phase_b<D>(c, t);
    if (c->mig) {
      if (has_nbr(c)) {
        mpm_status s = exchange_pair(c, MPM_XCHG_MIGRATE, mig_send_at(c, t, 0), mig_send_at(c, t, 1),
                                     mig_recv_at(c, t, 0), mig_recv_at(c, t, 1), c->mig_floats);
        if (s) return s;
      }
      forward_phase_c<D>(c, t);
    }
  }
  return MPM_OK;
}

// adjoint grid buffer of backward step t (double-buffered by step parity)
float4* agrid_of(mpm_ctx c, int t) { return (t & 1) ? c->agrid1 : c->agrid; }

// P2G^T variant: mass gradient on/off, material, block splitting for small problems
template <int D, bool MG, int MAT>
void launch_p2gT_v(mpm_ctx c, const KParams& P, const StepArgs& A, int na) {
  if (c->split) kx(c, k_p2g_adj<D, MG, MAT, true>, dim3(na), dim3(MPM_P2GT_THREADS), 0, P, A);
  else kx(c, k_p2g_adj<D, MG, MAT, false>, dim3(na), dim3(MPM_P2GT_THREADS), 0, P, A);
}
template <int D>
void launch_p2gT(mpm_ctx c, const KParams& P, const StepArgs& A, int na) {
  if (c->mass_grad) {
    if (P.material == 1) launch_p2gT_v<D, true, 1>(c, P, A, na);
    else launch_p2gT_v<D, true, 0>(c, P, A, na);
  } else {
    if (P.material == 1) launch_p2gT_v<D, false, 1>(c, P, A, na);
    else launch_p2gT_v<D, false, 0>(c, P, A, na);
  }
}

// backward step t = phase A ([zero,] G2P^T [, window pack]) | exchange | phase B ([unpack,]
// grid^T, P2G^T); the particle adjoint flows c->bcur -> c->bnxt
template <int D>
void backward_phase_a(mpm_ctx c, int t) {
  const KParams& P = c->P;
  StepArgs A = step_args(c, t);
  A.grid = agrid_of(c, t);
  A.gin = c->bcur;
  A.gout = c->bnxt;
  if (t == c->seg_end - 1)  // first backward step of a segment: prepare its buffer (later: by grid_T)
    launch(c, KI_ZERO, [&] { kx(c, k_zero_slots, dim3(c->n_sm * 4), dim3(256), 0, info_at(c, t), A.grid); });
  const int nbla = std::max(1, std::min(P.NBT, c->n_sm * c->occ_scatter_adj));
  launch(c, KI_G2PT, [&] {
    if (c->split) kx(c, k_block_scatter<D, true, 0, true>, dim3(nbla), dim3(kThreads), scatter_dyn_smem<D, true>(), P, A);
    else kx(c, k_block_scatter<D, true>, dim3(nbla), dim3(kThreads), scatter_dyn_smem<D, true>(), P, A);
  });
  if (has_nbr(c)) launch_band_pack(c, t, true, A.grid);
}

template <int D>
void backward_phase_b(mpm_ctx c, int t) {
  const KParams& P = c->P;
  StepArgs A = step_args(c, t);
  A.grid = agrid_of(c, t);
  A.gin = c->bcur;
  A.gout = c->bnxt;
  if (has_nbr(c)) launch_band_unpack(c, t, true, A.grid);
  if (MPM_GRIDT_FUSED && (c->split || MPM_GRIDT_FUSED >= 2)) {  // small problems: gridT inside P2G^T's tile staging; P2G^T
    A.info_prev = t > c->seg0 ? info_at(c, t - 1) : nullptr;  // also prepares step t-1's adjoint grid
    A.agrid_prev = agrid_of(c, t - 1);
  } else {
    launch(c, KI_GRIDT, [&] {
      kx(c, k_grid_adj<D>, dim3(c->n_sm * MPM_GRIDT_CTAS), dim3(256), 0, P, info_at(c, t), touch_at(c, t), c->arena, A.grid,
                                                         t > c->seg0 ? info_at(c, t - 1) : nullptr, agrid_of(c, t - 1));
    });
  }
  const int na = std::max(1, std::min(P.NBT, c->n_sm * c->occ_p2gT));
  launch(c, KI_P2GT, [&] { launch_p2gT<D>(c, P, A, na); });
  if (c->ctrl) {  // N1: controller adjoint of step t (needs this step's complete dL/da)
    const int KD = P.K * D;
    launch(c, KI_CTRLT, [&] {
      kx(c, k_ctrl_adj_param<D>, dim3(P.B), dim3(256), KD * sizeof(float), P, c->da, c->act, c->ctrl_W,
                                                                       c->gpre_tape + (size_t)t * P.B * KD,
                                                                       c->ctrl_gz, t);
    });
    launch(c, KI_CTRLT, [&] {
      kx(c, k_ctrl_adj_state<D>, dim3(c->n_sm * 4), dim3(256), 0, P, c->ctrl_gz, orig_at(c, t), c->prm, c->aid,
                                                              c->ctrl_Minv, c->bnxt);
    });
  }
}

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

// N1: group masses M[r][k] of the current particles -> 1/M (every group must be non-empty)
mpm_status ctrl_masses(mpm_ctx c) {
  const KParams& P = c->P;
  const int BK = P.B * P.K;
  CK(cudaMemsetAsync(c->ctrl_M, 0, BK * sizeof(float), c->stream));
  CK(cudaMemsetAsync(c->ctrl_n, 0, BK * sizeof(int), c->stream));
  launch(c, KI_MISC, [&] { k_ctrl_mass<<<c->n_sm * 2, 256, 0, c->stream>>>(P.NT, P.N, P.K, c->prm, c->aid, c->ctrl_M, c->ctrl_n); });
  std::vector<float> M(BK);
  std::vector<int> n(BK);
  CK(cudaMemcpyAsync(M.data(), c->ctrl_M, BK * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(n.data(), c->ctrl_n, BK * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < BK; ++i) {
    if (n[i] == 0 || !(M[i] > 0.f))
      return fail(c, MPM_ERR_INVALID_ARG, "controller: actuator group " + std::to_string(i % P.K) + " of rollout " +
                                              std::to_string(i / P.K) + " is empty");
    M[i] = 1.f / M[i];
  }
  CK(cudaMemcpyAsync(c->ctrl_Minv, M.data(), BK * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemsetAsync(c->ctrl_acc, 0, (size_t)BK * 2 * c->D * sizeof(float), c->stream));
  CK(cudaMemsetAsync(c->ctrl_cnt, 0, sizeof(int), c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return MPM_OK;
}

// (Re)allocate the tape's grid-slot arena for `per` slots per step (and the two per-step
// adjoint grids).  keep: copy the current arena's contents (the steps already on the tape keep
// their absolute slot numbers).  The old buffers are freed only once the new ones exist.
mpm_status alloc_arena(mpm_ctx c, long per, bool keep) {
  const size_t slots = (size_t)per * (size_t)(c->tape_cap + 1);
  float4 *na = nullptr, *ng0 = nullptr, *ng1 = nullptr;
  auto release = [&] {
    cudaFree(na);
    cudaFree(ng0);
    cudaFree(ng1);
    cudaGetLastError();
  };
  if (cudaMalloc(&na, slots * kCPB * sizeof(float4)) != cudaSuccess ||
      cudaMalloc(&ng0, (size_t)per * kCPB * sizeof(float4)) != cudaSuccess ||
      cudaMalloc(&ng1, (size_t)per * kCPB * sizeof(float4)) != cudaSuccess) {
    release();
    return fail(c, MPM_ERR_OOM, "grid-slot arena of " + std::to_string(slots * kCPB * sizeof(float4)) +
                                    " bytes: cudaMalloc failed");
  }
  drop_graphs(c);  // captured loops hold the old pointers
  if (c->arena) {
    if (keep) {
      CK(cudaMemcpyAsync(na, c->arena, c->arena_slots * kCPB * sizeof(float4), cudaMemcpyDeviceToDevice, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    for (void* old : {(void*)c->arena, (void*)c->agrid, (void*)c->agrid1}) {
      c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), old), c->allocs.end());
      cudaFree(old);
    }
  }
  for (void* q : {(void*)na, (void*)ng0, (void*)ng1}) c->allocs.push_back(q);
  c->arena = na;
  c->agrid = ng0;
  c->agrid1 = ng1;
  c->P.slots_per_step = (int)per;
  c->arena_slots = slots;
  c->P.arena_slots = (int)std::min<size_t>(slots, (size_t)0x7fffffff);
  return MPM_OK;
}

template <int D>
mpm_status do_set_state(mpm_ctx c, const float* x, const float* v, const float* F, const float* C,
                        const float* mass, const float* vol, const float* E, const float* nu,
                        const int32_t* aid) {
  const KParams& P = c->P;
  const size_t NT = P.NT, NU = c->NU;  // storage capacity, user-array length (equal outside migrating mode)
  c->seg0 = 0;  // a new rollout starts in tape slot 0
  c->res_end = 0;
  c->ck_valid = 0;
  // stage user arrays on the device (host or device pointers, UVA)
  float* sx = c->stage;
  float* sv = sx + NU * D;
  float* sF = sv + NU * D;
  float* sC = sF + NU * D * D;
  CK(cudaMemcpyAsync(sx, x, NU * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (v) CK(cudaMemcpyAsync(sv, v, NU * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (F) CK(cudaMemcpyAsync(sF, F, NU * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (C) CK(cudaMemcpyAsync(sC, C, NU * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  int n0 = (int)NT;
  if (c->mig) {
    // migrating slab mode: storage order 0 = the particles whose base_x the slab owns, in user
    // order (the binning decision of R17: fp32 x * res - 0.5, floor)
    std::vector<float> hx(NU * D);
    CK(cudaMemcpyAsync(hx.data(), sx, NU * D * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    std::vector<int> mem;
    for (size_t u = 0; u < NU; ++u) {
      const int bx = (int)floorf(hx[u * D] * P.fres - 0.5f);
      if (bx >= c->M.own_lo && bx < c->M.own_hi) mem.push_back((int)u);
    }
    if (mem.size() > NT)
      return fail(c, MPM_ERR_MIGRATE, "slab owns " + std::to_string(mem.size()) + " particles at t = 0, capacity " +
                                          std::to_string(NT) + " (config.n_particles)");
    n0 = (int)mem.size();
    CK(cudaMemcpyAsync(c->members, mem.data(), mem.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(orig_at(c, 0), c->members, mem.size() * sizeof(int), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(info_at(c, 0) + I_NSLOT, &n0, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));  // n0, mem are host locals
  }
  launch(c, KI_MISC, [&] {
    k_user_to_soa<D><<<grid1d(std::max(n0, 1)), 256, 0, c->stream>>>(P, sx, v ? sv : nullptr, F ? sF : nullptr,
                                                                       C ? sC : nullptr, state_at(c, 0),
                                                                       c->mig ? c->members : nullptr, n0);
  });
  float* pm = sC + NU * D * D;
  float* pv = pm + NU;
  CK(cudaMemcpyAsync(pm, mass, NU * sizeof(float), cudaMemcpyDefault, c->stream));
  CK(cudaMemcpyAsync(pv, vol, NU * sizeof(float), cudaMemcpyDefault, c->stream));
  CK(cudaMemcpyAsync(c->E, E, NU * sizeof(float), cudaMemcpyDefault, c->stream));
  CK(cudaMemcpyAsync(c->nu, nu, NU * sizeof(float), cudaMemcpyDefault, c->stream));
  if (aid) CK(cudaMemcpyAsync(c->aid, aid, NU * sizeof(int), cudaMemcpyDefault, c->stream));
  else CK(cudaMemsetAsync(c->aid, 0xff, NU * sizeof(int), c->stream));
  CK(cudaMemsetAsync(c->dbad, 0, sizeof(int), c->stream));
  launch(c, KI_MISC, [&] { k_params<<<grid1d(NU), 256, 0, c->stream>>>((int)NU, pm, pv, c->E, c->nu, c->prm, c->dbad); });
  CK(cudaMemsetAsync(c->err, 0, sizeof(ErrLatch), c->stream));
  CK(cudaMemsetAsync(c->cnt, 0, (size_t)P.NBT * sizeof(int), c->stream));
  launch_keys<D>(c, 0);
  if (c->ck) {  // N2: checkpoint 0 = the initial state
    CK(cudaMemcpyAsync(ck_state_of(c, 0), state_at(c, 0), recf(c) * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(ck_orig_of(c, 0), orig_at(c, 0), NT * sizeof(int), cudaMemcpyDeviceToDevice, c->stream));
    c->ck_valid = 1;
  }
  // grid-slot capacity per step: config.grid_slots, or automatic -- twice the touched blocks
  // of this initial state (re-sized on every set_state whose body needs more; grown during a
  // rollout that spreads beyond it, see mpm_forward)
  if (c->arena == nullptr || c->cfg.grid_slots <= 0) {
    launch(c, KI_MISC, [&] {
      if (c->cfg.fuse_g2p2g) kx(c, k_scan_a<D, true>, dim3(c->n_tiles), dim3(kScanTile), 0, P, c->cnt, c->bflag, c->tile_sums);
      else kx(c, k_scan_a<D>, dim3(c->n_tiles), dim3(kScanTile), 0, P, c->cnt, c->bflag, c->tile_sums);
    });
    std::vector<int3> ts(c->n_tiles);
    CK(cudaMemcpyAsync(ts.data(), c->tile_sums, ts.size() * sizeof(int3), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    long touched = 0;
    for (auto& q : ts) touched += q.z;
    const long per = c->cfg.grid_slots > 0 ? c->cfg.grid_slots
                                            : std::min<long>(P.NBT, 2 * touched + 64L * P.B + 64);
    if (c->arena == nullptr || per > c->P.slots_per_step) {
      mpm_status s = alloc_arena(c, per, false);
      if (s) return s;
    }
  }
  CK(cudaMemsetAsync(c->dmu, 0, NU * sizeof(float), c->stream));
  CK(cudaMemsetAsync(c->dlam, 0, NU * sizeof(float), c->stream));
  mpm_status s = sync_and_check(c, "set_state");
  int bad = 0;
  CK(cudaMemcpy(&bad, c->dbad, sizeof(int), cudaMemcpyDeviceToHost));
  if (s) return s;
  if (bad) return fail(c, MPM_ERR_INVALID_ARG, "parameters out of range (need mass > 0, vol > 0, E > 0, 0 <= nu < 0.5)");
  if (c->ctrl) {  // new particles: new group masses
    s = ctrl_masses(c);
    if (s) {
      c->ctrl = false;
      return s;
    }
  }
  c->tape_len = 0;
  c->has_state = true;
  c->has_grad = false;
  c->poisoned = false;
  return MPM_OK;
}

// A step loop can be a replayed graph when its launches depend on (direction, start, length)
// only: no host synchronisation or NCCL inside (no slab neighbours, no checkpoint segments),
// no per-launch profiling events, a non-legacy stream.  At least two steps: the binning scan's
// tile flags carry the epoch of the last scan, and a graph whose first and last scan are the
// same launch could read its own stale flags on the next replay.
constexpr size_t kGraphCache = 16;  // CUDA-graph executables kept per context (LRU)

bool graphs_ok(mpm_ctx c, int n) {
  return c->graphs && c->stream && !c->profiling && !has_nbr(c) && !has_xchg(c) && !c->mig && c->ck == 0 && n >= 2;
}

// Run body() -- which launches a step loop and advances the host state -- directly, or
// capture it into a graph on first use and replay it after.  The replay applies the host
// effects a capture records: the launch count and the scan epochs (later scans take fresh
// epochs, never one baked into a graph).  `after` restores the rest of the host state.
template <class F, class G>
mpm_status run_graphed(mpm_ctx c, int dir, int t0, int n, F&& body, G&& after) {
  if (!graphs_ok(c, n)) return body();
  for (size_t i = 0; i < c->gcache.size(); ++i)
    if (c->gcache[i].dir == dir && c->gcache[i].t0 == t0 && c->gcache[i].n == n) {
      std::rotate(c->gcache.begin() + i, c->gcache.begin() + i + 1, c->gcache.end());  // most recent last
      const auto& g = c->gcache.back();
      c->launches += g.launches;
      c->scan_epoch += g.epochs;
      after();
      CK(cudaGraphLaunch(g.exec, c->stream));
      return MPM_OK;
    }
  const int64_t l0 = c->launches;
  const unsigned e0 = c->scan_epoch;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  mpm_status s = body();
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
  cudaGraphExec_t exec = nullptr;
  if (!s && e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (s || e != cudaSuccess) {
    // body() advanced the host state (tape end, fused-grid step, adjoint buffers, counters)
    // for launches that never ran: undo the counters and refuse further steps until
    // mpm_set_state rebuilds a consistent context
    cudaGetLastError();
    c->launches = l0;
    c->scan_epoch = e0;
    c->poisoned = true;
    return s ? s : cuda_fail(c, e, "graph capture / instantiate (context reset required: mpm_set_state)");
  }
  // bounded cache: keep the kGraphCache most recent (direction, start, length) executables
  if (c->gcache.size() >= kGraphCache) {
    cudaStreamSynchronize(c->stream);
    cudaGraphExecDestroy(c->gcache.front().exec);
    c->gcache.erase(c->gcache.begin());
  }
  c->gcache.push_back({dir, t0, n, exec, c->launches - l0, c->scan_epoch - e0});
  CK(cudaGraphLaunch(exec, c->stream));
  return MPM_OK;
}

template <int D>
mpm_status do_forward(mpm_ctx c, int n) {
  const int t0 = c->tape_len;
  mpm_status s = run_graphed(
      c, 0, t0, n, [&] { return forward_range<D>(c, t0, t0 + n); },
      [&] {  // forward_range's host effects (checkpoint-free: seg0 is unchanged)
        c->res_end = t0 + n;
        c->fused_grid = -1;
      });
  if (s) return s;
  s = sync_and_check(c, "forward");
  if (s) return s;
  c->tape_len += n;
  return MPM_OK;
}

// N4: additive seed of state t into the adjoint buffer g, if registered
template <int D>
void add_step_seed(mpm_ctx c, int t, float* g) {
  auto it = c->seeds.find(t);
  if (it == c->seeds.end()) return;
  const size_t NT = c->P.NT;
  const float* b = it->second;
  const size_t NU = c->NU;  // seeds are user arrays
  launch(c, KI_MISC, [&] {
    kx(c, k_seed<D>, dim3(grid1d(NT)), dim3(256), 0, c->P, orig_at(c, t), b, b + NU * D, b + 2 * NU * D,
                                                  b + 2 * NU * D + NU * D * D, g, 1, nslot_at(c, t));
  });
}

// stage the terminal seed (user order AoS -> storage order T) and clear the accumulators
template <int D>
mpm_status backward_begin(mpm_ctx c, const float* gx, const float* gv, const float* gF, const float* gC) {
  const KParams& P = c->P;
  const size_t NT = P.NT, NU = c->NU;
  const int T = c->tape_len;
  float* sx = c->stage;
  float* sv = sx + NU * D;
  float* sF = sv + NU * D;
  float* sC = sF + NU * D * D;
  if (gx) CK(cudaMemcpyAsync(sx, gx, NU * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (gv) CK(cudaMemcpyAsync(sv, gv, NU * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (gF) CK(cudaMemcpyAsync(sF, gF, NU * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (gC) CK(cudaMemcpyAsync(sC, gC, NU * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  c->bcur = c->gA;
  c->bnxt = c->gB;
  launch(c, KI_MISC, [&] {
    kx(c, k_seed<D>, dim3(grid1d(NT)), dim3(256), 0, P, orig_at(c, T), gx ? sx : nullptr, gv ? sv : nullptr,
                                                  gF ? sF : nullptr, gC ? sC : nullptr, c->bcur, 0, nslot_at(c, T));
  });
  add_step_seed<D>(c, T, c->bcur);
  CK(cudaMemsetAsync(c->dmu, 0, NU * sizeof(float), c->stream));
  CK(cudaMemsetAsync(c->dlam, 0, NU * sizeof(float), c->stream));
  CK(cudaMemsetAsync(c->dmass, 0, NU * sizeof(float), c->stream));
  CK(cudaMemsetAsync(c->da, 0, (size_t)P.B * P.T * std::max(P.K, 1) * D * sizeof(float), c->stream));
  return MPM_OK;
}

template <int D>
void backward_step_end(mpm_ctx c, int t) {
  add_step_seed<D>(c, t, c->bnxt);
  std::swap(c->bcur, c->bnxt);
}

// gradient w.r.t. state 0 is in bcur (storage order 0 = user order); controller parameter
// gradients reduced over steps and rollouts
mpm_status backward_finish(mpm_ctx c) {
  if (c->bcur != c->gA)
    CK(cudaMemcpyAsync(c->gA, c->bcur, recf(c) * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
  if (c->ctrl) {
    const int T = c->tape_len;
    launch(c, KI_CTRLT, [&] {
      if (c->D == 3)
        k_ctrl_adj_reduce<3><<<c->n_sm, 128, 0, c->stream>>>(c->P, T, c->gpre_tape, c->ztape, c->ctrl_W, c->ctrl_gW,
                                                            c->ctrl_gb, c->ctrl_gt);
      else
        k_ctrl_adj_reduce<2><<<c->n_sm, 128, 0, c->stream>>>(c->P, T, c->gpre_tape, c->ztape, c->ctrl_W, c->ctrl_gW,
                                                            c->ctrl_gb, c->ctrl_gt);
    });
  }
  return MPM_OK;
}

size_t da_count(mpm_ctx c) { return (size_t)c->P.B * c->P.T * std::max(c->P.K, 1) * c->D; }

// N2: make checkpoint i (step i k) the first slot of the tape and recompute the keys of its state
template <int D>
void restore_checkpoint(mpm_ctx c, int i) {
  const size_t bs = recf(c) * sizeof(float), bo = NTs(c) * sizeof(int);
  c->seg0 = i * c->ck;
  c->res_end = c->seg0;
  cudaMemcpyAsync(c->tape_state, ck_state_of(c, i), bs, cudaMemcpyDeviceToDevice, c->stream);
  cudaMemcpyAsync(c->tape_orig, ck_orig_of(c, i), bo, cudaMemcpyDeviceToDevice, c->stream);
  cudaMemsetAsync(c->cnt, 0, (size_t)c->P.NBT * sizeof(int), c->stream);
  launch_keys<D>(c, c->seg0);
}

template <int D>
mpm_status do_backward(mpm_ctx c, const float* gx, const float* gv, const float* gF, const float* gC) {
  mpm_status s = backward_begin<D>(c, gx, gv, gF, gC);
  if (s) return s;
  c->seg_end = c->tape_len;  // the current segment [seg0, tape_len) is on the tape
  for (;;) {
    float* const b0 = c->bcur;
    float* const b1 = c->bnxt;
    const int steps = c->seg_end - c->seg0;
    s = run_graphed(
        c, 1, c->seg0, steps,
        [&]() -> mpm_status {
          for (int t = c->seg_end - 1; t >= c->seg0; --t) {
            if (c->mig && has_nbr(c)) {  // reverse migration of the adjoint of state t+1
              backward_mig_pack<D>(c, t);
              mpm_status q = exchange_pair(c, MPM_XCHG_MIGRATE_ADJ, c->rev_send[0], c->rev_send[1], c->rev_recv[0],
                                           c->rev_recv[1], rev_floats(c));
              if (q) return q;
              backward_mig_unpack<D>(c, t);
            }
            backward_phase_a<D>(c, t);
            if (has_nbr(c)) {
              mpm_status q = exchange_nccl(c);
              if (q) return q;
            }
            backward_phase_b<D>(c, t);
            backward_step_end<D>(c, t);
          }
          return MPM_OK;
        },
        [&] {  // the adjoint buffers swap once per step
          c->bcur = (steps & 1) ? b1 : b0;
          c->bnxt = (steps & 1) ? b0 : b1;
        });
    if (s) return s;
    if (c->seg0 == 0) break;
    // N2: recompute the previous segment from its checkpoint, then continue the reverse pass
    const int end = c->seg0;
    restore_checkpoint<D>(c, (end - 1) / c->ck);
    s = forward_range<D>(c, c->seg0, end);
    if (s) return s;
    c->seg_end = end;
    // the carried adjoint is in the storage order of the evicted run's state `end`
    // (= checkpoint end / k); map it to the recomputed order of that state
    const int NT = (int)NTs(c);
    launch(c, KI_MISC, [&] { k_invert_perm<<<grid1d(NT), 256, 0, c->stream>>>(NT, orig_at(c, end), c->scratch); });
    launch(c, KI_MISC, [&] {
      k_remap_adjoint<<<grid1d(NT), 256, 0, c->stream>>>(NT, c->S, ck_orig_of(c, end / c->ck), c->scratch, c->bcur,
                                                         c->bnxt);
    });
    std::swap(c->bcur, c->bnxt);
  }
  s = backward_finish(c);
  if (s) return s;
  if (c->slab && has_xchg(c)) {
    // slab mode: the actuation is shared by all slabs; migrating mode: a particle's dL/dmu,
    // dL/dlam, dL/dm collect on whichever slab simulated each step
    if (c->P.K > 0 && (s = allreduce_sum(c, c->da, da_count(c)))) return s;
    if (c->mig) {
      if ((s = allreduce_sum(c, c->dmu, c->NU))) return s;
      if ((s = allreduce_sum(c, c->dlam, c->NU))) return s;
      if (c->mass_grad && (s = allreduce_sum(c, c->dmass, c->NU))) return s;
    }
  }
  s = sync_and_check(c, "backward");
  if (s) return s;
  c->has_grad = true;
  c->mass_grad_valid = c->mass_grad;
  c->ctrl_grad_valid = c->ctrl;
  return MPM_OK;
}

template <int D>
mpm_status do_get_state(mpm_ctx c, int t, float* x, float* v, float* F, float* C) {
  const size_t NT = c->P.NT, NU = c->NU;
  float* sx = c->stage;
  float* sv = sx + NU * D;
  float* sF = sv + NU * D;
  float* sC = sF + NU * D * D;
  if (c->mig)  // this slab writes its own particles; zeros elsewhere (the sum over slabs is the body)
    CK(cudaMemsetAsync(sx, 0, NU * (2 * D + 2 * D * D) * sizeof(float), c->stream));
  launch(c, KI_MISC, [&] {
    k_soa_to_user<D><<<grid1d(NT), 256, 0, c->stream>>>(c->P, orig_at(c, t), state_at(c, t), sx, sv, sF, sC, 1,
                                                         nslot_at(c, t), c->mig ? state_at(c, t) : nullptr, c->M);
  });
  if (x) CK(cudaMemcpyAsync(x, sx, NU * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (v) CK(cudaMemcpyAsync(v, sv, NU * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (F) CK(cudaMemcpyAsync(F, sF, NU * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (C) CK(cudaMemcpyAsync(C, sC, NU * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  return sync_and_check(c, "get_state");
}

template <int D>
mpm_status do_grad(mpm_ctx c, float* dx0, float* dv0, float* dF0, float* dC0, float* dE, float* dnu, float* da) {
  const KParams& P = c->P;
  const size_t NT = P.NT, NU = c->NU;
  float* sx = c->stage;
  float* sv = sx + NU * D;
  float* sF = sv + NU * D;
  float* sC = sF + NU * D * D;
  float* sE = sC + NU * D * D;
  float* sn = sE + NU;
  if (c->mig) {  // storage order 0 = the members; zeros for the other slabs' particles
    CK(cudaMemsetAsync(sx, 0, NU * (2 * D + 2 * D * D) * sizeof(float), c->stream));
    launch(c, KI_MISC, [&] {
      k_soa_to_user<D><<<grid1d(NT), 256, 0, c->stream>>>(P, orig_at(c, 0), c->gA, sx, sv, sF, sC, 0, nslot_at(c, 0));
    });
  } else {
    launch(c, KI_MISC, [&] { k_soa_to_user<D><<<grid1d(NT), 256, 0, c->stream>>>(P, nullptr, c->gA, sx, sv, sF, sC, 0); });
  }
  launch(c, KI_MISC, [&] { k_finalize_params<<<grid1d(NU), 256, 0, c->stream>>>((int)NU, c->E, c->nu, c->dmu, c->dlam, sE, sn); });
  if (dx0) CK(cudaMemcpyAsync(dx0, sx, NU * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (dv0) CK(cudaMemcpyAsync(dv0, sv, NU * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (dF0) CK(cudaMemcpyAsync(dF0, sF, NU * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (dC0) CK(cudaMemcpyAsync(dC0, sC, NU * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (dE) CK(cudaMemcpyAsync(dE, sE, NU * sizeof(float), cudaMemcpyDefault, c->stream));
  if (dnu) CK(cudaMemcpyAsync(dnu, sn, NU * sizeof(float), cudaMemcpyDefault, c->stream));
  if (da && P.K > 0)
    CK(cudaMemcpyAsync(da, c->da, (size_t)P.B * P.T * P.K * D * sizeof(float), cudaMemcpyDefault, c->stream));
  return sync_and_check(c, "grad");
}

// N2: make state t resident on the tape (restore the nearest checkpoint at or before t and
// recompute forward to t); no-op when it already is.  Requires t <= tape_len.
template <int D>
mpm_status bring_to_tape(mpm_ctx c, int t) {
  if (on_tape(c, t)) return MPM_OK;
  if (!c->ck) return fail(c, MPM_ERR_CALL_ORDER, "step not on the tape");
  const int i = std::min(t / c->ck, c->ck_valid - 1);
  restore_checkpoint<D>(c, i);
  mpm_status s = forward_range<D>(c, c->seg0, t);
  if (s) return s;
  return sync_and_check(c, "checkpoint recompute");
}

template <int D>
mpm_status do_rewind(mpm_ctx c, int t) {
  CK(cudaMemsetAsync(c->err, 0, sizeof(ErrLatch), c->stream));
  if (!on_tape(c, t)) {
    mpm_status s = bring_to_tape<D>(c, t);
    if (s) return s;
  }
  CK(cudaMemsetAsync(c->cnt, 0, (size_t)c->P.NBT * sizeof(int), c->stream));
  launch_keys<D>(c, t);
  mpm_status s = sync_and_check(c, "rewind");
  if (s) return s;
  c->tape_len = t;
  c->poisoned = false;
  return MPM_OK;
}

}  // namespace

namespace {
mpm_status group_check(mpm_ctx* cs, int32_t n) {
  if (!cs || n < 1) return MPM_ERR_INVALID_ARG;
  for (int i = 0; i < n; ++i)
    if (!cs[i]) return MPM_ERR_INVALID_ARG;
  mpm_ctx c0 = cs[0];
  for (int i = 0; i < n; ++i) {
    mpm_ctx c = cs[i];
    if (!c->has_state) return fail(c, MPM_ERR_CALL_ORDER, "group call before mpm_set_state");
    if (c->poisoned) return fail(c, MPM_ERR_CALL_ORDER, "context poisoned by an earlier error; call mpm_set_state");
    if (c->comm) return fail(c, MPM_ERR_CALL_ORDER, "context has a communicator; use mpm_forward/mpm_backward");
    if (c->cfg.device != c0->cfg.device || c->stream != c0->stream || c->D != c0->D || c->P.res != c0->P.res ||
        c->tape_len != c0->tape_len || c->mig != c0->mig || c->cfg.fuse_g2p2g != c0->cfg.fuse_g2p2g ||
        c->ctrl != c0->ctrl ||
        (c->mig && (c->NU != c0->NU || c->M.mig_cap != c0->M.mig_cap)))
      return fail(c, MPM_ERR_INVALID_ARG, "group contexts need one device, one stream, equal dim/res/tape length, "
                                          "the same slab mode and the same fuse_g2p2g / controller setting");
    if (c->transport) return fail(c, MPM_ERR_CALL_ORDER, "context has a transport; use mpm_forward/mpm_backward");
    if (n > 1 && !c->slab) return fail(c, MPM_ERR_INVALID_ARG, "group contexts need mpm_set_slab");
    if (c->ck) return fail(c, MPM_ERR_INVALID_ARG, "group calls do not support checkpoint_every");
    if (c->slab) {
      const bool want_left = i > 0, want_right = i + 1 < n;
      if (c->left != want_left || c->right != want_right || (i + 1 < n && (c->x_hi != cs[i + 1]->x_lo ||
                                                                        c->halo != cs[i + 1]->halo)))
        return fail(c, MPM_ERR_INVALID_ARG, "group contexts must be adjacent slabs in x order with equal halo");
    }
  }
  return MPM_OK;
}

template <int D>
mpm_status group_forward(mpm_ctx* cs, int32_t n, int32_t steps) {
  const int t_end = cs[0]->tape_len + steps;
  for (int i = 0; i < n; ++i) cs[i]->fused_grid = -1;
  for (int k = 0; k < steps && fuse_on(cs[0]); ++k) {  // fused forward, windows summed between launches
    const int t = cs[0]->tape_len + k;
    bool built = false, next = false;
    for (int i = 0; i < n; ++i) built = fused_part_a<D>(cs[i], t, t_end);
    if (built && n > 1) {
      mpm_status s = exchange_local(cs, n);
      if (s) return s;
    }
    for (int i = 0; i < n; ++i) next = fused_part_b<D>(cs[i], t, t_end, built);
    if (next && n > 1) {
      mpm_status s = exchange_local(cs, n);
      if (s) return s;
      for (int i = 0; i < n; ++i) launch_band_unpack(cs[i], t + 1, false, cs[i]->arena);
    }
  }
  for (int k = 0; k < steps && !fuse_on(cs[0]); ++k) {
    const int t = cs[0]->tape_len + k;
    for (int i = 0; i < n; ++i) forward_phase_a<D>(cs[i], t);
    if (n > 1) {
      mpm_status s = exchange_local(cs, n);
      if (s) return s;
    }
    for (int i = 0; i < n; ++i) forward_phase_b<D>(cs[i], t);
    if (cs[0]->mig) {
      if (n > 1) {
        mpm_status s = exchange_local_mig(cs, n, t);
        if (s) return s;
      }
      for (int i = 0; i < n; ++i) forward_phase_c<D>(cs[i], t);
    }
  }
  mpm_status first = MPM_OK;
  for (int i = 0; i < n; ++i) {
    mpm_status s = sync_and_check(cs[i], "group forward");
    if (s && !first) first = s;
  }
  if (first) return first;
  for (int i = 0; i < n; ++i) cs[i]->tape_len += steps;
  return MPM_OK;
}

template <int D>
mpm_status group_backward(mpm_ctx* cs, int32_t n, const float* const* gx, const float* const* gv,
                          const float* const* gF, const float* const* gC) {
  for (int i = 0; i < n; ++i) {
    mpm_status s = backward_begin<D>(cs[i], gx ? gx[i] : nullptr, gv ? gv[i] : nullptr, gF ? gF[i] : nullptr,
                                     gC ? gC[i] : nullptr);
    if (s) return s;
  }
  for (int i = 0; i < n; ++i) cs[i]->seg_end = cs[i]->tape_len;
  for (int t = cs[0]->tape_len - 1; t >= 0; --t) {
    if (cs[0]->mig && n > 1) {  // reverse migration of the adjoint of state t+1
      for (int i = 0; i < n; ++i) backward_mig_pack<D>(cs[i], t);
      mpm_status s = exchange_local_rev(cs, n);
      if (s) return s;
      for (int i = 0; i < n; ++i) backward_mig_unpack<D>(cs[i], t);
    }
    for (int i = 0; i < n; ++i) backward_phase_a<D>(cs[i], t);
    if (n > 1) {
      mpm_status s = exchange_local(cs, n);
      if (s) return s;
    }
    for (int i = 0; i < n; ++i) {
      backward_phase_b<D>(cs[i], t);
      backward_step_end<D>(cs[i], t);
    }
  }
  for (int i = 0; i < n; ++i) {
    mpm_status s = backward_finish(cs[i]);
    if (s) return s;
  }
  mpm_ctx c = cs[0];
  // the actuation is shared by all slabs; in migrating mode a particle's dL/dmu, dL/dlam, dL/dm
  // collect on whichever slab simulated each step: every context gets the sums
  auto sum_all = [&](float* mpm_ctx_s::*field, size_t m) -> mpm_status {
    for (int i = 1; i < n; ++i)
      launch(c, KI_MISC, [&] { k_add_inplace<<<c->n_sm, 256, 0, c->stream>>>(m, c->*field, cs[i]->*field); });
    for (int i = 1; i < n; ++i)
      CK(cudaMemcpyAsync(cs[i]->*field, c->*field, m * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
    return MPM_OK;
  };
  if (n > 1) {
    mpm_status s = MPM_OK;
    if (c->P.K > 0 && (s = sum_all(&mpm_ctx_s::da, da_count(c)))) return s;
    if (c->mig) {
      if ((s = sum_all(&mpm_ctx_s::dmu, c->NU))) return s;
      if ((s = sum_all(&mpm_ctx_s::dlam, c->NU))) return s;
      if (c->mass_grad && (s = sum_all(&mpm_ctx_s::dmass, c->NU))) return s;
    }
  }
  mpm_status first = MPM_OK;
  for (int i = 0; i < n; ++i) {
    mpm_status s = sync_and_check(cs[i], "group backward");
    if (s && !first) first = s;
  }
  if (first) return first;
  for (int i = 0; i < n; ++i) {
    cs[i]->has_grad = true;
    cs[i]->mass_grad_valid = cs[i]->mass_grad;
    cs[i]->ctrl_grad_valid = cs[i]->ctrl;
  }
  return MPM_OK;
}
}  // namespace

// =====================================================================================
// ABI
// =====================================================================================
extern "C" {

mpm_status mpm_create(const mpm_config* cfg, mpm_ctx* out) {
  g_create_error.clear();
  if (!cfg || !out) {
    g_create_error = "mpm_create: null config or output pointer";
    return MPM_ERR_INVALID_ARG;
  }
  *out = nullptr;
  mpm_ctx c = new mpm_ctx_s();
  c->cfg = *cfg;
  const mpm_config& k = *cfg;
  auto bad = [&](const char* why) {
    g_create_error = why;
    delete c;
    return MPM_ERR_INVALID_ARG;
  };
  if (k.dim != 2 && k.dim != 3) return bad("dim must be 2 or 3");
  const int BB = k.dim == 3 ? 4 : 8;
  if (!is_pow2(k.res) || k.res < 16 || k.res > 4096) return bad("res must be a power of two in [16, 4096]");
  if (k.batch < 1 || k.n_particles < 1 || k.n_particles >= (1 << 25)) return bad("batch >= 1 and 1 <= n_particles < 2^25 required");
  if ((long long)k.batch * k.n_particles >= (1LL << 31)) return bad("batch * n_particles must be < 2^31");
  if (k.max_steps < 1) return bad("max_steps >= 1 required");
  if (k.material != 0 && k.material != 1) return bad("material must be 0 (neo-Hookean) or 1 (fixed-corotated)");
  if (k.checkpoint_every < 0 || k.checkpoint_every > k.max_steps) return bad("0 <= checkpoint_every <= max_steps required");
  if (k.fuse_g2p2g != 0 && k.fuse_g2p2g != 1) return bad("fuse_g2p2g must be 0 or 1");
  if (k.n_actuators < 0 || k.n_actuators > 64) return bad("n_actuators in [0, 64]");
  if (!(k.dt > 0.f)) return bad("dt > 0 required");
  if (k.bound < 0 || 2 * k.bound >= k.res) return bad("0 <= bound and 2*bound < res required");
  long long nbpa = k.res / BB, nb = 1;
  for (int a = 0; a < k.dim; ++a) nb *= nbpa;
  if (nb * k.batch >= (1LL << 31) / kCPB) return bad("too many grid blocks (batch * (res/Bb)^dim)");
  cudaError_t e = cudaSetDevice(k.device);
  if (e != cudaSuccess) {
    g_create_error = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
    delete c;
    return MPM_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, k.device);
  c->stream = (cudaStream_t)k.stream;
  if (const char* e = getenv("MPM_PDL")) c->pdl = atoi(e) != 0;
  c->D = k.dim;
  c->S = 2 * k.dim + 2 * k.dim * k.dim;
  KParams& P = c->P;
  P.res = k.res;
  P.B = k.batch;
  P.N = k.n_particles;
  P.NT = k.batch * k.n_particles;
  P.nbpa = (int)nbpa;
  P.nb = (int)nb;
  P.NBT = (int)(nb * k.batch);
  P.K = k.n_actuators;
  P.T = k.max_steps;
  P.dt = k.dt;
  P.dx = 1.0f / (float)k.res;
  P.fres = (float)k.res;
  for (int a = 0; a < 3; ++a) P.g[a] = (a < k.dim) ? k.gravity[a] : 0.f;
  P.bound = k.bound;
  for (int a = 0; a < 6; ++a) P.fric[a] = k.friction[a];
  P.act_s = k.act_strength;
  P.slab_lo = 0;
  P.slab_hi = k.res - 3;
  c->NU = (size_t)k.batch * k.n_particles;
  P.material = k.material;
  c->n_tiles = (P.NBT + kScanTile - 1) / kScanTile;
  // fewer than ~400 particles per gather CTA slot: too few occupied blocks to fill the GPU
  c->split = (long long)P.NT < 400LL * c->n_sm * 4;
  int occ = 0;
  // dynamic shared memory of the block-tile scatter (payload buffer) above the 48 KB default
  cudaFuncSetAttribute(k_block_scatter<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, scatter_dyn_smem<3, false>());
  cudaFuncSetAttribute(k_block_scatter<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, scatter_dyn_smem<3, true>());
  cudaFuncSetAttribute(k_block_scatter<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, scatter_dyn_smem<2, false>());
  cudaFuncSetAttribute(k_block_scatter<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, scatter_dyn_smem<2, true>());
  cudaFuncSetAttribute(k_block_scatter<3, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, scatter_dyn_smem<3, false>());
  cudaFuncSetAttribute(k_block_scatter<2, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, scatter_dyn_smem<2, false>());
  cudaFuncSetAttribute(k_block_scatter<3, true, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, scatter_dyn_smem<3, true>());
  cudaFuncSetAttribute(k_block_scatter<2, true, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, scatter_dyn_smem<2, true>());
  if (k.dim == 3) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_block_scatter<3, false>, kThreads, scatter_dyn_smem<3, false>());
    c->occ_scatter = std::max(1, occ);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_block_scatter<3, true>, kThreads, scatter_dyn_smem<3, true>());
    c->occ_scatter_adj = std::max(1, occ);
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_block_scatter<2, false>, kThreads, scatter_dyn_smem<2, false>());
    c->occ_scatter = std::max(1, occ);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_block_scatter<2, true>, kThreads, scatter_dyn_smem<2, true>());
    c->occ_scatter_adj = std::max(1, occ);
  }
  {  // NEXT N2 fused forward: payload buffer in dynamic shared memory
#define FA(D, MAT, SORT)                                                                                         \
  cudaFuncSetAttribute(k_g2p2g<D, MAT, SORT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, fuse_dyn_smem<D>()); \
  cudaFuncSetAttribute(k_g2p2g<D, MAT, SORT, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, fuse_dyn_smem<D>())
    FA(3, 0, false); FA(3, 0, true); FA(3, 1, false); FA(3, 1, true);
    FA(2, 0, false); FA(2, 0, true); FA(2, 1, false); FA(2, 1, true);
#undef FA
    if (k.dim == 3) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_g2p2g<3, 0, true, true>, kThreads, fuse_dyn_smem<3>());
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_g2p2g<2, 0, true, true>, kThreads, fuse_dyn_smem<2>());
    c->occ_fuse = std::max(1, occ);
  }
  if (k.dim == 3) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_g2p<3>, kThreads, 0);
    c->occ_g2p = std::max(1, occ);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_p2g_adj<3, false>, MPM_P2GT_THREADS, 0);
    c->occ_p2gT = std::max(1, occ);
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_g2p<2>, kThreads, 0);
    c->occ_g2p = std::max(1, occ);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_p2g_adj<2, false>, MPM_P2GT_THREADS, 0);
    c->occ_p2gT = std::max(1, occ);
  }

  const size_t NT = P.NT, T = k.max_steps, S = c->S, D = k.dim;
  // N2: with checkpoint_every = k the tape holds one k-step segment, plus T/k + 1 checkpoints
  c->ck = k.checkpoint_every;
  c->tape_cap = c->ck ? c->ck : k.max_steps;
  c->n_ck = c->ck ? k.max_steps / c->ck + 1 : 0;
  const size_t TC = c->tape_cap;
  mpm_status s = MPM_OK;
#define AL(ptr, n) \
  if (!s) s = dalloc(c, &c->ptr, (n))
  const size_t RF = rec_floats((int)S, NT);  // one particle-record buffer (AoSoA: padded)
  AL(tape_state, (TC + 1) * RF);
  AL(tape_perm, TC * NT);
  AL(tape_orig, (TC + 1) * NT);
  AL(tape_bs, TC * (size_t)(P.NBT + 1));
  AL(tape_slot, TC * (size_t)P.NBT);
  AL(tape_occ, TC * (size_t)P.NBT);
  AL(tape_touch, TC * (size_t)P.NBT);
  AL(info, (TC + 1) * kInfo);
  if (c->ck) {
    AL(ck_state, (size_t)c->n_ck * RF);
    AL(ck_orig, (size_t)c->n_ck * NT);
  }
  AL(key, NT);
  AL(cnt, (size_t)P.NBT);
  AL(tmp_pk, NT);
  AL(scratch, NT);
  AL(hist2, (size_t)P.NBT);
  AL(tile_sums, (size_t)c->n_tiles);
  AL(scan.flag, (size_t)c->n_tiles);
  AL(scan.agg, (size_t)c->n_tiles);
  AL(scan.incl, (size_t)c->n_tiles);
  AL(scan.ticket, 1);
  AL(bflag, (size_t)P.NBT);
  AL(err, 1);
  AL(dbad, 1);
  AL(prm, NT);
  AL(aid, NT);
  AL(E, NT);
  AL(nu, NT);
  AL(act, (size_t)P.B * T * std::max(P.K, 1) * D);
  AL(gA, RF);
  AL(gB, RF);
  AL(dmu, NT);
  AL(dlam, NT);
  AL(dmass, NT);
  AL(da, (size_t)P.B * T * std::max(P.K, 1) * D);
  AL(stage, NT * (2 * D + 2 * D * D + 2));
#undef AL
  if (s) {
    g_create_error = c->last_error;
    mpm_destroy(c);
    return s;
  }
  cudaMemset(c->err, 0, sizeof(ErrLatch));
  cudaMemset(c->scan.flag, 0, (size_t)c->n_tiles * sizeof(unsigned));
  cudaMemset(c->scan.ticket, 0, sizeof(unsigned long long));
  cudaMemset(c->cnt, 0, (size_t)P.NBT * sizeof(int));
  cudaMemset(c->act, 0, (size_t)P.B * T * std::max(P.K, 1) * D * sizeof(float));
  cudaMemset(c->info, 0, (TC + 1) * kInfo * sizeof(int));
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    g_create_error = std::string("device initialisation: ") + cudaGetErrorString(e);
    mpm_destroy(c);
    return MPM_ERR_CUDA;
  }
  *out = c;
  return MPM_OK;
}

void mpm_destroy(mpm_ctx c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  else cudaDeviceSynchronize();
  if (c->comm) nccl_api()->CommDestroy(c->comm);
  if (c->host_stage) cudaFreeHost(c->host_stage);
  for (void* p : c->allocs) cudaFree(p);
  for (auto& kv : c->seeds) cudaFree(kv.second);
  for (auto& p : c->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  drop_graphs(c);
  delete c;
}

mpm_status mpm_set_state(mpm_ctx c, const float* x, const float* v, const float* F, const float* C,
                         const float* mass, const float* vol, const float* E, const float* nu,
                         const int32_t* aid) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (!x || !mass || !vol || !E || !nu) return fail(c, MPM_ERR_INVALID_ARG, "x, mass, vol, E, nu are required");
  cudaSetDevice(c->cfg.device);
  return c->D == 3 ? do_set_state<3>(c, x, v, F, C, mass, vol, E, nu, aid)
                   : do_set_state<2>(c, x, v, F, C, mass, vol, E, nu, aid);
}

mpm_status mpm_set_actuation(mpm_ctx c, const float* a) {
  if (!c || !a) return MPM_ERR_INVALID_ARG;
  if (c->P.K == 0) return MPM_OK;
  cudaSetDevice(c->cfg.device);
  size_t n = (size_t)c->P.B * c->P.T * c->P.K * c->D;
  CK(cudaMemcpyAsync(c->act, a, n * sizeof(float), cudaMemcpyDefault, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->has_act = true;
  return MPM_OK;
}

mpm_status mpm_forward(mpm_ctx c, int32_t n) {
  if (!c || n < 0) return MPM_ERR_INVALID_ARG;
  if (!c->has_state) return fail(c, MPM_ERR_CALL_ORDER, "mpm_forward before mpm_set_state");
  if (c->poisoned) return fail(c, MPM_ERR_CALL_ORDER, "context poisoned by an earlier error; call mpm_set_state");
  if (c->tape_len + n > c->cfg.max_steps) return fail(c, MPM_ERR_TAPE_FULL, "forward beyond max_steps");
  if (has_nbr(c) && !has_xchg(c))
    return fail(c, MPM_ERR_CALL_ORDER, "slab context with neighbours: call mpm_comm_init / mpm_set_transport, or use mpm_group_forward");
  cudaSetDevice(c->cfg.device);
  c->has_grad = false;
  if (!on_tape(c, c->tape_len)) {  // N2: the tape end was evicted by a checkpointed backward
    mpm_status s = c->D == 3 ? bring_to_tape<3>(c, c->tape_len) : bring_to_tape<2>(c, c->tape_len);
    if (s) return s;
  }
  const int t_end = c->tape_len + n;
  for (;;) {
    mpm_status s = c->D == 3 ? do_forward<3>(c, t_end - c->tape_len) : do_forward<2>(c, t_end - c->tape_len);
    // automatic capacity (config.grid_slots = 0): a body that spread beyond the grid-slot arena
    // sized at set_state.  Steps before the latched one are intact (the overflow is detected by
    // the binning scan of the grid being built, before anything is written into it); grow the
    // arena x2 keeping them, rewind to that step and carry on.  Not in slab mode with a
    // communicator (the ranks would diverge) nor with checkpoints (the step may not be resident).
    const bool growable = s == MPM_ERR_TAPE_FULL && c->cfg.grid_slots <= 0 && !c->comm && c->ck == 0 &&
                          c->P.slots_per_step < c->P.NBT && c->latch_step >= c->seg0 && c->latch_step < t_end;
    if (!growable) return s;
    const int t_fail = c->latch_step;
    s = alloc_arena(c, std::min<long>(c->P.NBT, 2L * c->P.slots_per_step), true);
    if (s) return s;
    c->poisoned = false;
    c->tape_len = std::max(c->tape_len, t_fail);  // do_forward advanced nothing on failure
    s = c->D == 3 ? do_rewind<3>(c, t_fail) : do_rewind<2>(c, t_fail);
    if (s) return s;
  }
}

int32_t mpm_tape_length(mpm_ctx c) { return c ? c->tape_len : -1; }

mpm_status mpm_rewind(mpm_ctx c, int32_t t) {
  if (!c || t < 0) return MPM_ERR_INVALID_ARG;
  if (!c->has_state || t > c->tape_len) return fail(c, MPM_ERR_CALL_ORDER, "rewind beyond the tape");
  cudaSetDevice(c->cfg.device);
  c->has_grad = false;
  return c->D == 3 ? do_rewind<3>(c, t) : do_rewind<2>(c, t);
}

mpm_status mpm_get_state(mpm_ctx c, int32_t t, float* x, float* v, float* F, float* C) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (!c->has_state || t < 0 || t > c->tape_len) return fail(c, MPM_ERR_CALL_ORDER, "step not on the tape");
  cudaSetDevice(c->cfg.device);
  if (!on_tape(c, t)) {  // N2: recompute from the nearest checkpoint
    mpm_status s = c->D == 3 ? bring_to_tape<3>(c, t) : bring_to_tape<2>(c, t);
    if (s) return s;
  }
  return c->D == 3 ? do_get_state<3>(c, t, x, v, F, C) : do_get_state<2>(c, t, x, v, F, C);
}

mpm_status mpm_backward(mpm_ctx c, const float* gx, const float* gv, const float* gF, const float* gC) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (!c->has_state) return fail(c, MPM_ERR_CALL_ORDER, "mpm_backward before mpm_set_state");
  if (c->poisoned) return fail(c, MPM_ERR_CALL_ORDER, "context poisoned by an earlier error; call mpm_set_state");
  if (has_nbr(c) && !has_xchg(c))
    return fail(c, MPM_ERR_CALL_ORDER, "slab context with neighbours: call mpm_comm_init / mpm_set_transport, or use mpm_group_backward");
  cudaSetDevice(c->cfg.device);
  if (!on_tape(c, c->tape_len)) {  // N2: bring the last segment back
    mpm_status s = c->D == 3 ? bring_to_tape<3>(c, c->tape_len) : bring_to_tape<2>(c, c->tape_len);
    if (s) return s;
  }
  return c->D == 3 ? do_backward<3>(c, gx, gv, gF, gC) : do_backward<2>(c, gx, gv, gF, gC);
}

mpm_status mpm_grad(mpm_ctx c, float* dx0, float* dv0, float* dF0, float* dC0, float* dE, float* dnu, float* da) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (!c->has_grad) return fail(c, MPM_ERR_CALL_ORDER, "mpm_grad before mpm_backward");
  cudaSetDevice(c->cfg.device);
  return c->D == 3 ? do_grad<3>(c, dx0, dv0, dF0, dC0, dE, dnu, da) : do_grad<2>(c, dx0, dv0, dF0, dC0, dE, dnu, da);
}

const char* mpm_last_error(mpm_ctx c) {
  if (c) return c->last_error.c_str();
  return g_create_error.empty() ? "null context" : g_create_error.c_str();
}

mpm_status mpm_get_binning(mpm_ctx c, int32_t t, float* x_store, int32_t* orig, int32_t* keyo, int32_t* perm,
                           int32_t* block_start) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (!c->has_state || t < 0 || t >= c->tape_len || t < c->seg0 || t + 1 > c->res_end)
    return fail(c, MPM_ERR_CALL_ORDER, "step not on the tape (checkpointed: not resident)");
  cudaSetDevice(c->cfg.device);
  const KParams& P = c->P;
  const size_t NT = P.NT;
  const int D = c->D;
  if (x_store) {
    // record buffer -> [NT][D] storage order
    std::vector<float> h(recf(c));
    CK(cudaMemcpyAsync(h.data(), state_at(c, t), h.size() * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    std::vector<float> o((size_t)D * NT);
    for (size_t j = 0; j < NT; ++j)
      for (int a = 0; a < D; ++a) o[j * D + a] = h[rixs(c->S, a, (int)j, NT)];
    CK(cudaMemcpy(x_store, o.data(), o.size() * sizeof(float), cudaMemcpyDefault));
  }
  if (orig) CK(cudaMemcpyAsync(orig, orig_at(c, t), NT * sizeof(int), cudaMemcpyDefault, c->stream));
  if (perm) CK(cudaMemcpyAsync(perm, perm_at(c, t), NT * sizeof(int), cudaMemcpyDefault, c->stream));
  if (block_start) CK(cudaMemcpyAsync(block_start, bs_at(c, t), (P.NBT + 1) * sizeof(int), cudaMemcpyDefault, c->stream));
  if (keyo) {
    // keys of storage order t: recompute from the stored positions (same device code as the step)
    int* tmp = c->scratch;
    if (D == 3)
      k_init_keys<3><<<grid1d(NT), 256, 0, c->stream>>>(P, state_at(c, t), tmp, c->hist2, nullptr, c->err, nslot_at(c, t), c->M);
    else
      k_init_keys<2><<<grid1d(NT), 256, 0, c->stream>>>(P, state_at(c, t), tmp, c->hist2, nullptr, c->err, nslot_at(c, t), c->M);
    CK(cudaMemcpyAsync(keyo, tmp, NT * sizeof(int), cudaMemcpyDefault, c->stream));
  }
  return sync_and_check(c, "get_binning");
}

mpm_status mpm_get_grid(mpm_ctx c, int32_t t, float* m, float* vbar) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (!c->has_state || t < 0 || t >= c->tape_len || t < c->seg0 || t + 1 > c->res_end)
    return fail(c, MPM_ERR_CALL_ORDER, "step not on the tape (checkpointed: not resident)");
  cudaSetDevice(c->cfg.device);
  const KParams& P = c->P;
  size_t nn = 1;
  for (int a = 0; a < c->D; ++a) nn *= P.res;
  nn *= P.B;
  float *dm = nullptr, *dv = nullptr;
  struct Free {  // temporaries released on every return path
    float** p[2];
    ~Free() {
      for (float** q : p) cudaFree(*q);
    }
  } guard{{&dm, &dv}};
  mpm_status s = MPM_OK;
  CK(cudaMalloc(&dm, nn * sizeof(float)));
  CK(cudaMalloc(&dv, nn * c->D * sizeof(float)));
  CK(cudaMemsetAsync(dm, 0, nn * sizeof(float), c->stream));
  CK(cudaMemsetAsync(dv, 0, nn * c->D * sizeof(float), c->stream));
  if (c->D == 3)
    k_dense_grid<3><<<c->n_sm * 8, 256, 0, c->stream>>>(P, info_at(c, t), touch_at(c, t), c->arena, dm, dv);
  else
    k_dense_grid<2><<<c->n_sm * 8, 256, 0, c->stream>>>(P, info_at(c, t), touch_at(c, t), c->arena, dm, dv);
  if (m) CK(cudaMemcpyAsync(m, dm, nn * sizeof(float), cudaMemcpyDefault, c->stream));
  if (vbar) CK(cudaMemcpyAsync(vbar, dv, nn * c->D * sizeof(float), cudaMemcpyDefault, c->stream));
  s = sync_and_check(c, "get_grid");
  return s;
}

mpm_status mpm_get_step_info(mpm_ctx c, int32_t t, int32_t out[3]) {
  if (!c || !out) return MPM_ERR_INVALID_ARG;
  if (!c->has_state || t < 0 || t >= c->tape_len || t < c->seg0 || t + 1 > c->res_end)
    return fail(c, MPM_ERR_CALL_ORDER, "step not on the tape (checkpointed: not resident)");
  cudaSetDevice(c->cfg.device);
  int h[kInfo];
  CK(cudaMemcpy(h, info_at(c, t), sizeof(h), cudaMemcpyDeviceToHost));
  out[0] = h[I_NOCC];
  out[1] = h[I_NTOUCH];
  out[2] = h[I_BASE];
  return MPM_OK;
}

mpm_status mpm_set_profiling(mpm_ctx c, int32_t on) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (!on && c->profiling) {
    cudaStreamSynchronize(c->stream);
    drain_profile(c);
  }
  c->profiling = on != 0;
  if (on) {
    for (int i = 0; i < KI_COUNT; ++i) {
      c->prof_ms[i] = 0;
      c->prof_n[i] = 0;
    }
  }
  return MPM_OK;
}

mpm_status mpm_get_profile(mpm_ctx c, int32_t* n_kernels, float* ms, int64_t* launches, char* names, int32_t names_len) {
  if (!c || !n_kernels) return MPM_ERR_INVALID_ARG;
  cudaStreamSynchronize(c->stream);
  drain_profile(c);
  int n = std::min<int>(*n_kernels, KI_COUNT);
  if (*n_kernels <= 0) n = KI_COUNT;
  std::string all;
  for (int i = 0; i < KI_COUNT; ++i) {
    if (i < n) {
      if (ms) ms[i] = (float)c->prof_ms[i];
      if (launches) launches[i] = c->prof_n[i];
    }
    all += kKernelNames[i];
    if (i + 1 < KI_COUNT) all += ";";
  }
  *n_kernels = KI_COUNT;
  if (names && names_len > 0) {
    strncpy(names, all.c_str(), names_len - 1);
    names[names_len - 1] = 0;
  }
  return MPM_OK;
}

int64_t mpm_launch_count(mpm_ctx c) { return c ? c->launches : -1; }

mpm_status mpm_set_graphs(mpm_ctx c, int32_t on) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (on && !c->stream) return fail(c, MPM_ERR_INVALID_ARG, "CUDA graphs need config.stream (not the legacy default stream)");
  cudaSetDevice(c->cfg.device);
  if (!on) drop_graphs(c);
  c->graphs = on != 0;
  return MPM_OK;
}

mpm_status mpm_add_seed(mpm_ctx c, int32_t t, const float* dLdx, const float* dLdv, const float* dLdF,
                        const float* dLdC) {
  if (!c || t < 0 || t > c->cfg.max_steps) return MPM_ERR_INVALID_ARG;
  cudaSetDevice(c->cfg.device);
  const size_t NT = c->NU, D = c->D;  // a seed is a user array
  const size_t n = NT * (2 * D + 2 * D * D);
  float*& b = c->seeds[t];
  if (!b) {
    drop_graphs(c);  // a new seed step: the backward graphs do not launch its k_seed
    mpm_status s = dalloc(c, &b, n);
    if (s) {
      c->seeds.erase(t);
      return s;
    }
    c->allocs.pop_back();  // owned by the seed map (freed by mpm_clear_seeds / destroy)
    CK(cudaMemsetAsync(b, 0, n * sizeof(float), c->stream));
  }
  const float* src[4] = {dLdx, dLdv, dLdF, dLdC};
  const size_t off[4] = {0, NT * D, 2 * NT * D, 2 * NT * D + NT * D * D};
  const size_t len[4] = {NT * D, NT * D, NT * D * D, NT * D * D};
  for (int i = 0; i < 4; ++i)
    if (src[i]) CK(cudaMemcpyAsync(b + off[i], src[i], len[i] * sizeof(float), cudaMemcpyDefault, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return MPM_OK;
}

mpm_status mpm_clear_seeds(mpm_ctx c) {
  if (!c) return MPM_ERR_INVALID_ARG;
  cudaSetDevice(c->cfg.device);
  cudaStreamSynchronize(c->stream);
  drop_graphs(c);
  for (auto& kv : c->seeds) cudaFree(kv.second);
  c->seeds.clear();
  return MPM_OK;
}

mpm_status mpm_enable_mass_grad(mpm_ctx c, int32_t on) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if ((on != 0) != c->mass_grad) drop_graphs(c);  // P2G^T variant baked into backward graphs
  c->mass_grad = on != 0;
  c->mass_grad_valid = false;
  return MPM_OK;
}

mpm_status mpm_grad_mass(mpm_ctx c, float* dmass) {
  if (!c || !dmass) return MPM_ERR_INVALID_ARG;
  if (!c->has_grad || !c->mass_grad_valid)
    return fail(c, MPM_ERR_CALL_ORDER, "mpm_grad_mass needs mpm_enable_mass_grad(1) before mpm_backward");
  cudaSetDevice(c->cfg.device);
  CK(cudaMemcpyAsync(dmass, c->dmass, c->NU * sizeof(float), cudaMemcpyDefault, c->stream));
  return sync_and_check(c, "grad_mass");
}

// ---- slab mode ----

mpm_status mpm_set_slab(mpm_ctx c, int32_t x_lo, int32_t x_hi, int32_t halo) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (c->has_state) return fail(c, MPM_ERR_CALL_ORDER, "mpm_set_slab must precede mpm_set_state");
  if (c->slab) return fail(c, MPM_ERR_INVALID_ARG, "slab already set");
  const KParams& P = c->P;
  const int BB = c->D == 3 ? Dim<3>::BB : Dim<2>::BB, res = P.res;
  if (P.B != 1) return fail(c, MPM_ERR_INVALID_ARG, "slab mode needs batch == 1");
  if (halo < 1) return fail(c, MPM_ERR_INVALID_ARG, "halo_blocks >= 1 required");
  if (x_lo < 0 || x_hi > res || x_lo >= x_hi || x_lo % BB || x_hi % BB)
    return fail(c, MPM_ERR_INVALID_ARG, "need 0 <= x_lo < x_hi <= res, both multiples of the block size");
  const bool left = x_lo > 0, right = x_hi < res;
  const int hw = halo * BB;
  if ((left || right) && x_hi - x_lo < 2 * hw)
    return fail(c, MPM_ERR_INVALID_ARG, "slab narrower than two halo windows (2 * halo_blocks * block size)");
  if ((left && x_lo < hw) || (right && x_hi + hw > res))
    return fail(c, MPM_ERR_INVALID_ARG, "halo window outside the domain");
  cudaSetDevice(c->cfg.device);
  const int plane = P.nb / P.nbpa;  // blocks per block-plane
  c->band_blocks = 2 * halo * plane;
  c->gb_lo = (x_lo / BB - halo) * plane;
  c->gb_hi = (x_hi / BB - halo) * plane;
  if (left || right) {
    const size_t n = (size_t)c->band_blocks * kCPB;
    mpm_status s = dalloc(c, &c->send_lo, n);
    if (!s) s = dalloc(c, &c->send_hi, n);
    if (!s) s = dalloc(c, &c->recv_lo, n);
    if (!s) s = dalloc(c, &c->recv_hi, n);
    if (s) return s;
  }
  c->slab = true;
  c->left = left;
  c->right = right;
  c->x_lo = x_lo;
  c->x_hi = x_hi;
  c->halo = halo;
  c->P.slab_lo = left ? x_lo - hw : 0;
  c->P.slab_hi = right ? std::min(x_hi + hw - 3, res - 3) : res - 3;
  return MPM_OK;
}

mpm_status mpm_set_slab_migrating(mpm_ctx c, int32_t x_lo, int32_t x_hi, int32_t halo, int32_t n_global,
                                  int32_t mig_cap) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (c->cfg.checkpoint_every) return fail(c, MPM_ERR_INVALID_ARG, "migrating slab mode needs checkpoint_every = 0");
  if (c->ctrl) return fail(c, MPM_ERR_INVALID_ARG, "migrating slab mode does not support the controller");
  if (n_global < 1) return fail(c, MPM_ERR_INVALID_ARG, "n_global >= 1 required");
  if (mig_cap < 0) return fail(c, MPM_ERR_INVALID_ARG, "mig_cap >= 0 required");
  mpm_status s = mpm_set_slab(c, x_lo, x_hi, halo);
  if (s) return s;
  KParams& P = c->P;
  const int D = c->D;
  // ownership: base_x in [x_lo, x_hi) (the outer slabs also take what lies beyond; the domain
  // check rejects it); no drift bound
  P.slab_lo = 0;
  P.slab_hi = P.res - 3;
  c->M.migrate = 1;
  c->M.own_lo = c->left ? x_lo : INT32_MIN;
  c->M.own_hi = c->right ? x_hi : INT32_MAX;
  c->M.mig_cap = mig_cap > 0 ? mig_cap : std::max(1024, P.NT / 64);
  c->mig = true;
  c->NU = (size_t)n_global;
  c->mig_floats = Mig<3>::HDR + (size_t)c->M.mig_cap * (D == 3 ? Mig<3>::R : Mig<2>::R);
  // user-indexed arrays span the whole body now (the storage ones keep the capacity P.NT)
  auto realloc_user = [&](auto*& ptr, size_t count) -> mpm_status {
    c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), (void*)ptr), c->allocs.end());
    cudaFree(ptr);
    ptr = nullptr;
    return dalloc(c, &ptr, count);
  };
  const size_t NU = c->NU, TC = c->tape_cap;
  if (!s) s = realloc_user(c->prm, NU);
  if (!s) s = realloc_user(c->aid, NU);
  if (!s) s = realloc_user(c->E, NU);
  if (!s) s = realloc_user(c->nu, NU);
  if (!s) s = realloc_user(c->dmu, NU);
  if (!s) s = realloc_user(c->dlam, NU);
  if (!s) s = realloc_user(c->dmass, NU);
  if (!s) s = realloc_user(c->stage, NU * (2 * D + 2 * D * D + 2));
  if (!s) s = dalloc(c, &c->members, (size_t)P.NT);
  if (!s) s = dalloc(c, &c->mig_send_tape, TC * 2 * c->mig_floats);
  if (!s) s = dalloc(c, &c->mig_recv_tape, TC * 2 * c->mig_floats);
  for (int side = 0; side < 2 && !s; ++side) {
    s = dalloc(c, &c->rev_send[side], rev_floats(c));
    if (!s) s = dalloc(c, &c->rev_recv[side], rev_floats(c));
  }
  if (s) return s;
  CK(cudaMemset(c->mig_recv_tape, 0, TC * 2 * c->mig_floats * sizeof(float)));
  CK(cudaMemset(c->mig_send_tape, 0, TC * 2 * c->mig_floats * sizeof(float)));
  return MPM_OK;
}

mpm_status mpm_set_transport(mpm_ctx c, mpm_transport_fn fn, void* user) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (c->comm && fn) return fail(c, MPM_ERR_CALL_ORDER, "context already has an NCCL communicator");
  if (fn && !c->slab) return fail(c, MPM_ERR_CALL_ORDER, "mpm_set_transport needs mpm_set_slab first");
  drop_graphs(c);
  c->transport = fn;
  c->transport_user = user;
  return MPM_OK;
}

mpm_status mpm_comm_unique_id(char out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  if (!out) return MPM_ERR_INVALID_ARG;
  const NcclApi* N = nccl_api();
  if (!N) return MPM_ERR_COMM;
  ncclUniqueId id;
  if (N->GetUniqueId(&id) != ncclSuccess) return MPM_ERR_COMM;
  memcpy(out, &id, sizeof id);
  return MPM_OK;
}

mpm_status mpm_comm_init(mpm_ctx c, int32_t rank, int32_t world, const char id[128]) {
  if (!c || !id || world < 1 || rank < 0 || rank >= world) return MPM_ERR_INVALID_ARG;
  if (!c->slab) return fail(c, MPM_ERR_CALL_ORDER, "mpm_comm_init needs mpm_set_slab first");
  if (c->comm) return fail(c, MPM_ERR_CALL_ORDER, "communicator already initialised");
  if (c->transport) return fail(c, MPM_ERR_CALL_ORDER, "context has a transport callback");
  if ((c->left && rank == 0) || (c->right && rank == world - 1))
    return fail(c, MPM_ERR_INVALID_ARG, "ranks must be ordered by slab (left neighbour = rank - 1)");
  const NcclApi* N = nccl_api();
  if (!N) return fail(c, MPM_ERR_COMM, "libnccl.so.2 not found");
  cudaSetDevice(c->cfg.device);
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  ncclResult_t r = N->CommInitRank(&c->comm, world, uid, rank);
  if (r != ncclSuccess) {
    c->comm = nullptr;
    return fail(c, MPM_ERR_COMM, std::string("ncclCommInitRank: ") + N->GetErrorString(r));
  }
  c->rank = rank;
  c->world = world;
  return MPM_OK;
}

mpm_status mpm_group_forward(mpm_ctx* cs, int32_t n, int32_t steps) {
  mpm_status s = group_check(cs, n);
  if (s) return s;
  if (steps < 0) return MPM_ERR_INVALID_ARG;
  if (cs[0]->tape_len + steps > cs[0]->cfg.max_steps)
    return fail(cs[0], MPM_ERR_TAPE_FULL, "forward beyond max_steps");
  for (int i = 0; i < n; ++i)
    if (cs[i]->tape_len + steps > cs[i]->cfg.max_steps) return fail(cs[i], MPM_ERR_TAPE_FULL, "forward beyond max_steps");
  cudaSetDevice(cs[0]->cfg.device);
  for (int i = 0; i < n; ++i) cs[i]->has_grad = false;
  return cs[0]->D == 3 ? group_forward<3>(cs, n, steps) : group_forward<2>(cs, n, steps);
}

mpm_status mpm_group_backward(mpm_ctx* cs, int32_t n, const float* const* dLdx, const float* const* dLdv,
                              const float* const* dLdF, const float* const* dLdC) {
  mpm_status s = group_check(cs, n);
  if (s) return s;
  cudaSetDevice(cs[0]->cfg.device);
  return cs[0]->D == 3 ? group_backward<3>(cs, n, dLdx, dLdv, dLdF, dLdC)
                       : group_backward<2>(cs, n, dLdx, dLdv, dLdF, dLdC);
}

// ---- NEXT N1: closed-loop controller ----

mpm_status mpm_set_controller(mpm_ctx c, const float* W, const float* b, const float* target) {
  if (!c) return MPM_ERR_INVALID_ARG;
  cudaSetDevice(c->cfg.device);
  drop_graphs(c);  // the controller kernels (and P.nz) are baked into captured step loops
  if (!W) {
    c->ctrl = false;
    return MPM_OK;
  }
  if (!b || !target) return fail(c, MPM_ERR_INVALID_ARG, "W, b and target are required");
  if (!c->has_state) return fail(c, MPM_ERR_CALL_ORDER, "mpm_set_controller needs mpm_set_state first");
  KParams& P = c->P;
  const int D = c->D;
  if (P.K < 1) return fail(c, MPM_ERR_INVALID_ARG, "the controller needs n_actuators >= 1");
  if (has_nbr(c) || c->mig) return fail(c, MPM_ERR_INVALID_ARG, "the controller is not supported across slabs");
  const int KD = P.K * D, nz = D * (1 + 2 * P.K);
  const size_t T = c->cfg.max_steps;
  if (!c->ctrl_W) {
    mpm_status s = MPM_OK;
#define AL(ptr, n) \
  if (!s) s = dalloc(c, &c->ptr, (n))
    AL(ctrl_W, (size_t)KD * nz);
    AL(ctrl_b, KD);
    AL(ctrl_target, D);
    AL(ctrl_Minv, (size_t)P.B * P.K);
    AL(ctrl_M, (size_t)P.B * P.K);
    AL(ctrl_n, (size_t)P.B * P.K);
    AL(ctrl_acc, (size_t)P.B * P.K * 2 * D);
    AL(ctrl_cnt, 1);
    AL(ztape, T * P.B * nz);
    AL(gpre_tape, T * P.B * KD);
    AL(ctrl_gz, (size_t)P.B * nz);
    AL(ctrl_gW, (size_t)KD * nz);
    AL(ctrl_gb, KD);
    AL(ctrl_gt, D);
#undef AL
    if (s) return s;
  }
  P.nz = nz;
  CK(cudaMemcpyAsync(c->ctrl_W, W, (size_t)KD * nz * sizeof(float), cudaMemcpyDefault, c->stream));
  CK(cudaMemcpyAsync(c->ctrl_b, b, KD * sizeof(float), cudaMemcpyDefault, c->stream));
  CK(cudaMemcpyAsync(c->ctrl_target, target, D * sizeof(float), cudaMemcpyDefault, c->stream));
  mpm_status s = ctrl_masses(c);
  if (s) return s;
  c->ctrl = true;
  c->has_grad = false;
  return MPM_OK;
}

mpm_status mpm_grad_controller(mpm_ctx c, float* dW, float* db, float* dtarget) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (!c->has_grad || !c->ctrl_grad_valid)
    return fail(c, MPM_ERR_CALL_ORDER, "mpm_grad_controller needs a backward run with the controller on");
  cudaSetDevice(c->cfg.device);
  const int KD = c->P.K * c->D;
  if (dW) CK(cudaMemcpyAsync(dW, c->ctrl_gW, (size_t)KD * c->P.nz * sizeof(float), cudaMemcpyDefault, c->stream));
  if (db) CK(cudaMemcpyAsync(db, c->ctrl_gb, KD * sizeof(float), cudaMemcpyDefault, c->stream));
  if (dtarget) CK(cudaMemcpyAsync(dtarget, c->ctrl_gt, c->D * sizeof(float), cudaMemcpyDefault, c->stream));
  return sync_and_check(c, "grad_controller");
}

}  // extern "C"
