// mpm_api.cu -- C ABI + runtime of the B200-native differentiable MLS-MPM step.
// Declared in include/mpm.h.  Owns device memory, the tape (the paper's memo),
// the per-step launch schedule, the device error latch and per-kernel profiling.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/mpm.h"
#include "mpm_kernels.cuh"

using namespace mpm;

namespace {

enum KernelId {
  KI_SCAN_A, KI_SCAN_B, KI_SCAN_C, KI_SCATTER, KI_P2G, KI_GRID, KI_G2P,
  KI_ZERO, KI_G2PT, KI_GRIDT, KI_P2GT, KI_MISC, KI_COUNT
};
const char* kKernelNames[KI_COUNT] = {"scan_a", "scan_b", "scan_c",  "scatter", "p2g",  "grid_update",
                                      "g2p",    "zero_adj", "g2p_T", "grid_T", "p2g_T", "misc"};

struct PendingEvent {
  cudaEvent_t a, b;
  int kid;
};

}  // namespace

struct mpm_ctx_s {
  mpm_config cfg{};
  KParams P{};
  int D = 3, S = 24;
  cudaStream_t stream = nullptr;
  int n_sm = 148;
  int occ_scatter = 2, occ_scatter_adj = 2, occ_g2p = 2, occ_p2gT = 2;
  int tape_len = 0;
  bool has_state = false, has_act = false, has_grad = false, poisoned = false;
  std::string last_error;
  int64_t launches = 0;
  // tape
  float* tape_state = nullptr;
  int* tape_perm = nullptr;
  int* tape_orig = nullptr;
  int* tape_bs = nullptr;
  int* tape_slot = nullptr;
  int* tape_occ = nullptr;
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
  // profiling
  bool profiling = false;
  bool mass_grad = false;  // N3: compute dL/dm_p in P2G^T (opt-in)
  bool mass_grad_valid = false;
  std::vector<PendingEvent> pending;
  std::vector<cudaEvent_t> event_pool;
  double prof_ms[KI_COUNT] = {};
  int64_t prof_n[KI_COUNT] = {};
};

namespace {

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

size_t NTs(mpm_ctx c) { return (size_t)c->P.NT; }
float* state_at(mpm_ctx c, int t) { return c->tape_state + (size_t)t * c->S * NTs(c); }
int* perm_at(mpm_ctx c, int t) { return c->tape_perm + (size_t)t * NTs(c); }
int* orig_at(mpm_ctx c, int t) { return c->tape_orig + (size_t)t * NTs(c); }
int* bs_at(mpm_ctx c, int t) { return c->tape_bs + (size_t)t * (c->P.NBT + 1); }
int* slot_at(mpm_ctx c, int t) { return c->tape_slot + (size_t)t * c->P.NBT; }
int* occ_at(mpm_ctx c, int t) { return c->tape_occ + (size_t)t * c->P.NBT; }
int* touch_at(mpm_ctx c, int t) { return c->tape_touch + (size_t)t * c->P.NBT; }
int* info_at(mpm_ctx c, int t) { return c->info + (size_t)t * kInfo; }

int grid1d(size_t n, int bs = 256) { return (int)((n + bs - 1) / bs); }

// Read the device error latch (after a stream sync) and turn it into a status.
mpm_status check_latch(mpm_ctx c) {
  ErrLatch h{};
  cudaError_t e = cudaMemcpy(&h, c->err, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(c, e, "error latch readback");
  if (h.code == 0) return MPM_OK;
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
  launch(c, KI_MISC, [&] {
    k_init_keys<D><<<grid1d(P.NT), 256, 0, c->stream>>>(P, state_at(c, t), c->key, c->cnt,
                                                         t == 0 ? orig_at(c, 0) : c->scratch, c->err);
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

// binning tables of step t from the keys/histogram of state t
template <int D>
void launch_bin(mpm_ctx c, int t) {
  const KParams& P = c->P;
  launch(c, KI_SCAN_A, [&] { k_scan_a<D><<<c->n_tiles, kThreads, 0, c->stream>>>(P, c->cnt, c->bflag, c->tile_sums); });
  launch(c, KI_SCAN_B, [&] { k_scan_b<<<1, kThreads, 0, c->stream>>>(P, c->n_tiles, c->tile_sums, c->info, t, c->err); });
  launch(c, KI_SCAN_C, [&] {
    k_scan_c<<<c->n_tiles, kThreads, 0, c->stream>>>(P, c->bflag, c->tile_sums, info_at(c, t), bs_at(c, t),
                                                      slot_at(c, t), occ_at(c, t), touch_at(c, t));
  });
  launch(c, KI_SCATTER, [&] {
    k_scatter<<<grid1d(P.NT), 256, 0, c->stream>>>(P.NT, c->key, bs_at(c, t), c->cnt, c->tmp_pk, info_at(c, t), c->arena);
  });
}

template <int D>
void launch_forward_step(mpm_ctx c, int t) {
  const KParams& P = c->P;
  launch_bin<D>(c, t);
  StepArgs A = step_args(c, t);
  const int nblk = std::max(1, std::min(P.NBT, c->n_sm * c->occ_scatter));
  launch(c, KI_P2G, [&] { k_block_scatter<D, false><<<nblk, kThreads, scatter_dyn_smem<D, false>(), c->stream>>>(P, A); });
  const int ng = std::max(1, std::min(P.NBT, c->n_sm * c->occ_g2p));
  launch(c, KI_G2P, [&] { k_g2p<D><<<ng, kThreads, 0, c->stream>>>(P, A); });
}

// adjoint grid buffer of backward step t (double-buffered by step parity)
float4* agrid_of(mpm_ctx c, int t) { return (t & 1) ? c->agrid1 : c->agrid; }

template <int D>
void launch_backward_step(mpm_ctx c, int t, const float* gin, float* gout) {
  const KParams& P = c->P;
  StepArgs A = step_args(c, t);
  A.grid = agrid_of(c, t);
  A.gin = gin;
  A.gout = gout;

  const int nblk = std::max(1, std::min(P.NBT, c->n_sm * c->occ_scatter));
  if (t == c->tape_len - 1)  // first backward step: prepare its buffer (later steps: by grid_T)
    launch(c, KI_ZERO, [&] { k_zero_slots<<<c->n_sm * 4, 256, 0, c->stream>>>(info_at(c, t), A.grid); });
  const int nbla = std::max(1, std::min(P.NBT, c->n_sm * c->occ_scatter_adj));
  launch(c, KI_G2PT, [&] { k_block_scatter<D, true><<<nbla, kThreads, scatter_dyn_smem<D, true>(), c->stream>>>(P, A); });
  launch(c, KI_GRIDT, [&] {
    k_grid_adj<D><<<c->n_sm * 8, 256, 0, c->stream>>>(P, info_at(c, t), touch_at(c, t), c->arena, A.grid,
                                                       t > 0 ? info_at(c, t - 1) : nullptr, agrid_of(c, t - 1));
  });
  const int na = std::max(1, std::min(P.NBT, c->n_sm * c->occ_p2gT));
  if (c->mass_grad)
    launch(c, KI_P2GT, [&] { k_p2g_adj<D, true><<<na, MPM_P2GT_THREADS, 0, c->stream>>>(P, A); });
  else
    launch(c, KI_P2GT, [&] { k_p2g_adj<D, false><<<na, MPM_P2GT_THREADS, 0, c->stream>>>(P, A); });
}

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

template <int D>
mpm_status do_set_state(mpm_ctx c, const float* x, const float* v, const float* F, const float* C,
                        const float* mass, const float* vol, const float* E, const float* nu,
                        const int32_t* aid) {
  const KParams& P = c->P;
  const size_t NT = P.NT;
  // stage user arrays on the device (host or device pointers, UVA)
  float* sx = c->stage;
  float* sv = sx + NT * D;
  float* sF = sv + NT * D;
  float* sC = sF + NT * D * D;
  CK(cudaMemcpyAsync(sx, x, NT * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (v) CK(cudaMemcpyAsync(sv, v, NT * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (F) CK(cudaMemcpyAsync(sF, F, NT * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (C) CK(cudaMemcpyAsync(sC, C, NT * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  launch(c, KI_MISC, [&] {
    k_user_to_soa<D><<<grid1d(NT), 256, 0, c->stream>>>(P, sx, v ? sv : nullptr, F ? sF : nullptr,
                                                         C ? sC : nullptr, state_at(c, 0));
  });
  float* pm = sC + NT * D * D;
  float* pv = pm + NT;
  CK(cudaMemcpyAsync(pm, mass, NT * sizeof(float), cudaMemcpyDefault, c->stream));
  CK(cudaMemcpyAsync(pv, vol, NT * sizeof(float), cudaMemcpyDefault, c->stream));
  CK(cudaMemcpyAsync(c->E, E, NT * sizeof(float), cudaMemcpyDefault, c->stream));
  CK(cudaMemcpyAsync(c->nu, nu, NT * sizeof(float), cudaMemcpyDefault, c->stream));
  if (aid) CK(cudaMemcpyAsync(c->aid, aid, NT * sizeof(int), cudaMemcpyDefault, c->stream));
  else CK(cudaMemsetAsync(c->aid, 0xff, NT * sizeof(int), c->stream));
  CK(cudaMemsetAsync(c->dbad, 0, sizeof(int), c->stream));
  launch(c, KI_MISC, [&] { k_params<<<grid1d(NT), 256, 0, c->stream>>>((int)NT, pm, pv, c->E, c->nu, c->prm, c->dbad); });
  CK(cudaMemsetAsync(c->err, 0, sizeof(ErrLatch), c->stream));
  CK(cudaMemsetAsync(c->cnt, 0, (size_t)P.NBT * sizeof(int), c->stream));
  launch_keys<D>(c, 0);
  // automatic grid-slot capacity from the touched blocks of the initial state
  if (c->arena == nullptr) {
    launch(c, KI_SCAN_A, [&] { k_scan_a<D><<<c->n_tiles, kThreads, 0, c->stream>>>(P, c->cnt, c->bflag, c->tile_sums); });
    std::vector<int3> ts(c->n_tiles);
    CK(cudaMemcpyAsync(ts.data(), c->tile_sums, ts.size() * sizeof(int3), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    long touched = 0;
    for (auto& q : ts) touched += q.z;
    long per = c->cfg.grid_slots > 0 ? c->cfg.grid_slots
                                      : std::min<long>(P.NBT, 2 * touched + 64L * P.B + 64);
    c->P.slots_per_step = (int)per;
    c->arena_slots = (size_t)per * (size_t)(c->cfg.max_steps + 1);
    c->P.arena_slots = (int)std::min<size_t>(c->arena_slots, (size_t)0x7fffffff);
    mpm_status s = dalloc(c, &c->arena, c->arena_slots * kCPB);
    if (s) return s;
    s = dalloc(c, &c->agrid, (size_t)per * kCPB);
    if (s) return s;
    s = dalloc(c, &c->agrid1, (size_t)per * kCPB);
    if (s) return s;
  }
  CK(cudaMemsetAsync(c->dmu, 0, NT * sizeof(float), c->stream));
  CK(cudaMemsetAsync(c->dlam, 0, NT * sizeof(float), c->stream));
  mpm_status s = sync_and_check(c, "set_state");
  int bad = 0;
  CK(cudaMemcpy(&bad, c->dbad, sizeof(int), cudaMemcpyDeviceToHost));
  if (s) return s;
  if (bad) return fail(c, MPM_ERR_INVALID_ARG, "parameters out of range (need mass > 0, vol > 0, E > 0, 0 <= nu < 0.5)");
  c->tape_len = 0;
  c->has_state = true;
  c->has_grad = false;
  c->poisoned = false;
  return MPM_OK;
}

template <int D>
mpm_status do_forward(mpm_ctx c, int n) {
  for (int i = 0; i < n; ++i) launch_forward_step<D>(c, c->tape_len + i);
  mpm_status s = sync_and_check(c, "forward");
  if (s) return s;
  c->tape_len += n;
  return MPM_OK;
}

template <int D>
mpm_status do_backward(mpm_ctx c, const float* gx, const float* gv, const float* gF, const float* gC) {
  const KParams& P = c->P;
  const size_t NT = P.NT;
  const int T = c->tape_len;
  // stage seeds (user order AoS) then permute into storage order T
  float* sx = c->stage;
  float* sv = sx + NT * D;
  float* sF = sv + NT * D;
  float* sC = sF + NT * D * D;
  if (gx) CK(cudaMemcpyAsync(sx, gx, NT * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (gv) CK(cudaMemcpyAsync(sv, gv, NT * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (gF) CK(cudaMemcpyAsync(sF, gF, NT * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (gC) CK(cudaMemcpyAsync(sC, gC, NT * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  float* cur = c->gA;
  float* nxt = c->gB;
  launch(c, KI_MISC, [&] {
    k_seed<D><<<grid1d(NT), 256, 0, c->stream>>>(P, orig_at(c, T), gx ? sx : nullptr, gv ? sv : nullptr,
                                                  gF ? sF : nullptr, gC ? sC : nullptr, cur, 0);
  });
  auto add_step_seed = [&](int t, float* g) {  // N4: additive seed of state t, if registered
    auto it = c->seeds.find(t);
    if (it == c->seeds.end()) return;
    const float* b = it->second;
    launch(c, KI_MISC, [&] {
      k_seed<D><<<grid1d(NT), 256, 0, c->stream>>>(P, orig_at(c, t), b, b + NT * D, b + 2 * NT * D,
                                                    b + 2 * NT * D + NT * D * D, g, 1);
    });
  };
  add_step_seed(T, cur);
  CK(cudaMemsetAsync(c->dmu, 0, NT * sizeof(float), c->stream));
  CK(cudaMemsetAsync(c->dlam, 0, NT * sizeof(float), c->stream));
  CK(cudaMemsetAsync(c->dmass, 0, NT * sizeof(float), c->stream));
  CK(cudaMemsetAsync(c->da, 0, (size_t)P.B * P.T * std::max(P.K, 1) * D * sizeof(float), c->stream));
  for (int t = T - 1; t >= 0; --t) {
    launch_backward_step<D>(c, t, cur, nxt);
    add_step_seed(t, nxt);
    std::swap(cur, nxt);
  }
  // gradient w.r.t. state 0 now in `cur` (storage order 0 = user order)
  if (cur != c->gA) CK(cudaMemcpyAsync(c->gA, cur, (size_t)c->S * NT * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
  mpm_status s = sync_and_check(c, "backward");
  if (s) return s;
  c->has_grad = true;
  c->mass_grad_valid = c->mass_grad;
  return MPM_OK;
}

template <int D>
mpm_status do_get_state(mpm_ctx c, int t, float* x, float* v, float* F, float* C) {
  const size_t NT = c->P.NT;
  float* sx = c->stage;
  float* sv = sx + NT * D;
  float* sF = sv + NT * D;
  float* sC = sF + NT * D * D;
  launch(c, KI_MISC, [&] {
    k_soa_to_user<D><<<grid1d(NT), 256, 0, c->stream>>>(c->P, orig_at(c, t), state_at(c, t), sx, sv, sF, sC, 1);
  });
  if (x) CK(cudaMemcpyAsync(x, sx, NT * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (v) CK(cudaMemcpyAsync(v, sv, NT * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (F) CK(cudaMemcpyAsync(F, sF, NT * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (C) CK(cudaMemcpyAsync(C, sC, NT * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  return sync_and_check(c, "get_state");
}

template <int D>
mpm_status do_grad(mpm_ctx c, float* dx0, float* dv0, float* dF0, float* dC0, float* dE, float* dnu, float* da) {
  const KParams& P = c->P;
  const size_t NT = P.NT;
  float* sx = c->stage;
  float* sv = sx + NT * D;
  float* sF = sv + NT * D;
  float* sC = sF + NT * D * D;
  float* sE = sC + NT * D * D;
  float* sn = sE + NT;
  launch(c, KI_MISC, [&] { k_soa_to_user<D><<<grid1d(NT), 256, 0, c->stream>>>(P, nullptr, c->gA, sx, sv, sF, sC, 0); });
  launch(c, KI_MISC, [&] { k_finalize_params<<<grid1d(NT), 256, 0, c->stream>>>((int)NT, c->E, c->nu, c->dmu, c->dlam, sE, sn); });
  if (dx0) CK(cudaMemcpyAsync(dx0, sx, NT * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (dv0) CK(cudaMemcpyAsync(dv0, sv, NT * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (dF0) CK(cudaMemcpyAsync(dF0, sF, NT * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (dC0) CK(cudaMemcpyAsync(dC0, sC, NT * D * D * sizeof(float), cudaMemcpyDefault, c->stream));
  if (dE) CK(cudaMemcpyAsync(dE, sE, NT * sizeof(float), cudaMemcpyDefault, c->stream));
  if (dnu) CK(cudaMemcpyAsync(dnu, sn, NT * sizeof(float), cudaMemcpyDefault, c->stream));
  if (da && P.K > 0)
    CK(cudaMemcpyAsync(da, c->da, (size_t)P.B * P.T * P.K * D * sizeof(float), cudaMemcpyDefault, c->stream));
  return sync_and_check(c, "grad");
}

template <int D>
mpm_status do_rewind(mpm_ctx c, int t) {
  CK(cudaMemsetAsync(c->cnt, 0, (size_t)c->P.NBT * sizeof(int), c->stream));
  CK(cudaMemsetAsync(c->err, 0, sizeof(ErrLatch), c->stream));
  launch_keys<D>(c, t);
  mpm_status s = sync_and_check(c, "rewind");
  if (s) return s;
  c->tape_len = t;
  c->poisoned = false;
  return MPM_OK;
}

}  // namespace

// =====================================================================================
// ABI
// =====================================================================================
extern "C" {

mpm_status mpm_create(const mpm_config* cfg, mpm_ctx* out) {
  if (!cfg || !out) return MPM_ERR_INVALID_ARG;
  *out = nullptr;
  mpm_ctx c = new mpm_ctx_s();
  c->cfg = *cfg;
  const mpm_config& k = *cfg;
  auto bad = [&](const char* why) {
    c->last_error = why;
    delete c;
    return MPM_ERR_INVALID_ARG;
  };
  if (k.dim != 2 && k.dim != 3) return bad("dim must be 2 or 3");
  const int BB = k.dim == 3 ? 4 : 8;
  if (!is_pow2(k.res) || k.res < 16 || k.res > 4096) return bad("res must be a power of two in [16, 4096]");
  if (k.batch < 1 || k.n_particles < 1 || k.n_particles >= (1 << 25)) return bad("batch >= 1 and 1 <= n_particles < 2^25 required");
  if ((long long)k.batch * k.n_particles >= (1LL << 31)) return bad("batch * n_particles must be < 2^31");
  if (k.max_steps < 1) return bad("max_steps >= 1 required");
  if (k.n_actuators < 0 || k.n_actuators > 64) return bad("n_actuators in [0, 64]");
  if (!(k.dt > 0.f)) return bad("dt > 0 required");
  if (k.bound < 0 || 2 * k.bound >= k.res) return bad("0 <= bound and 2*bound < res required");
  long long nbpa = k.res / BB, nb = 1;
  for (int a = 0; a < k.dim; ++a) nb *= nbpa;
  if (nb * k.batch >= (1LL << 31) / kCPB) return bad("too many grid blocks (batch * (res/Bb)^dim)");
  cudaError_t e = cudaSetDevice(k.device);
  if (e != cudaSuccess) {
    c->last_error = cudaGetErrorString(e);
    delete c;
    return MPM_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, k.device);
  c->stream = (cudaStream_t)k.stream;
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
  c->n_tiles = (P.NBT + kScanTile - 1) / kScanTile;
  int occ = 0;
  // dynamic shared memory of the block-tile scatter (payload buffer) above the 48 KB default
  cudaFuncSetAttribute(k_block_scatter<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, scatter_dyn_smem<3, false>());
  cudaFuncSetAttribute(k_block_scatter<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, scatter_dyn_smem<3, true>());
  cudaFuncSetAttribute(k_block_scatter<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, scatter_dyn_smem<2, false>());
  cudaFuncSetAttribute(k_block_scatter<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, scatter_dyn_smem<2, true>());
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
  mpm_status s = MPM_OK;
#define AL(ptr, n) \
  if (!s) s = dalloc(c, &c->ptr, (n))
  AL(tape_state, (T + 1) * S * NT);
  AL(tape_perm, T * NT);
  AL(tape_orig, (T + 1) * NT);
  AL(tape_bs, T * (size_t)(P.NBT + 1));
  AL(tape_slot, T * (size_t)P.NBT);
  AL(tape_occ, T * (size_t)P.NBT);
  AL(tape_touch, T * (size_t)P.NBT);
  AL(info, (T + 1) * kInfo);
  AL(key, NT);
  AL(cnt, (size_t)P.NBT);
  AL(tmp_pk, NT);
  AL(scratch, NT);
  AL(hist2, (size_t)P.NBT);
  AL(tile_sums, (size_t)c->n_tiles);
  AL(bflag, (size_t)P.NBT);
  AL(err, 1);
  AL(dbad, 1);
  AL(prm, NT);
  AL(aid, NT);
  AL(E, NT);
  AL(nu, NT);
  AL(act, (size_t)P.B * T * std::max(P.K, 1) * D);
  AL(gA, S * NT);
  AL(gB, S * NT);
  AL(dmu, NT);
  AL(dlam, NT);
  AL(dmass, NT);
  AL(da, (size_t)P.B * T * std::max(P.K, 1) * D);
  AL(stage, NT * (2 * D + 2 * D * D + 2));
#undef AL
  if (s) {
    std::string why = c->last_error;
    mpm_destroy(c);
    return s;
  }
  cudaMemset(c->err, 0, sizeof(ErrLatch));
  cudaMemset(c->cnt, 0, (size_t)P.NBT * sizeof(int));
  cudaMemset(c->act, 0, (size_t)P.B * T * std::max(P.K, 1) * D * sizeof(float));
  cudaMemset(c->info, 0, (T + 1) * kInfo * sizeof(int));
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    c->last_error = cudaGetErrorString(e);
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
  for (void* p : c->allocs) cudaFree(p);
  for (auto& kv : c->seeds) cudaFree(kv.second);
  for (auto& p : c->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : c->event_pool) cudaEventDestroy(e);
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
  cudaSetDevice(c->cfg.device);
  c->has_grad = false;
  return c->D == 3 ? do_forward<3>(c, n) : do_forward<2>(c, n);
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
  return c->D == 3 ? do_get_state<3>(c, t, x, v, F, C) : do_get_state<2>(c, t, x, v, F, C);
}

mpm_status mpm_backward(mpm_ctx c, const float* gx, const float* gv, const float* gF, const float* gC) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (!c->has_state) return fail(c, MPM_ERR_CALL_ORDER, "mpm_backward before mpm_set_state");
  if (c->poisoned) return fail(c, MPM_ERR_CALL_ORDER, "context poisoned by an earlier error; call mpm_set_state");
  cudaSetDevice(c->cfg.device);
  return c->D == 3 ? do_backward<3>(c, gx, gv, gF, gC) : do_backward<2>(c, gx, gv, gF, gC);
}

mpm_status mpm_grad(mpm_ctx c, float* dx0, float* dv0, float* dF0, float* dC0, float* dE, float* dnu, float* da) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (!c->has_grad) return fail(c, MPM_ERR_CALL_ORDER, "mpm_grad before mpm_backward");
  cudaSetDevice(c->cfg.device);
  return c->D == 3 ? do_grad<3>(c, dx0, dv0, dF0, dC0, dE, dnu, da) : do_grad<2>(c, dx0, dv0, dF0, dC0, dE, dnu, da);
}

const char* mpm_last_error(mpm_ctx c) { return c ? c->last_error.c_str() : "null context"; }

mpm_status mpm_get_binning(mpm_ctx c, int32_t t, float* x_store, int32_t* orig, int32_t* keyo, int32_t* perm,
                           int32_t* block_start) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (!c->has_state || t < 0 || t >= c->tape_len) return fail(c, MPM_ERR_CALL_ORDER, "step not on the tape");
  cudaSetDevice(c->cfg.device);
  const KParams& P = c->P;
  const size_t NT = P.NT;
  const int D = c->D;
  if (x_store) {
    // SoA -> [NT][D] storage order
    std::vector<float> h((size_t)D * NT);
    CK(cudaMemcpyAsync(h.data(), state_at(c, t), h.size() * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    std::vector<float> o((size_t)D * NT);
    for (size_t j = 0; j < NT; ++j)
      for (int a = 0; a < D; ++a) o[j * D + a] = h[a * NT + j];
    CK(cudaMemcpy(x_store, o.data(), o.size() * sizeof(float), cudaMemcpyDefault));
  }
  if (orig) CK(cudaMemcpyAsync(orig, orig_at(c, t), NT * sizeof(int), cudaMemcpyDefault, c->stream));
  if (perm) CK(cudaMemcpyAsync(perm, perm_at(c, t), NT * sizeof(int), cudaMemcpyDefault, c->stream));
  if (block_start) CK(cudaMemcpyAsync(block_start, bs_at(c, t), (P.NBT + 1) * sizeof(int), cudaMemcpyDefault, c->stream));
  if (keyo) {
    // keys of storage order t: recompute from the stored positions (same device code as the step)
    int* tmp = c->scratch;
    if (D == 3)
      k_init_keys<3><<<grid1d(NT), 256, 0, c->stream>>>(P, state_at(c, t), tmp, c->hist2, reinterpret_cast<int*>(c->tmp_pk), c->err);
    else
      k_init_keys<2><<<grid1d(NT), 256, 0, c->stream>>>(P, state_at(c, t), tmp, c->hist2, reinterpret_cast<int*>(c->tmp_pk), c->err);
    CK(cudaMemcpyAsync(keyo, tmp, NT * sizeof(int), cudaMemcpyDefault, c->stream));
  }
  return sync_and_check(c, "get_binning");
}

mpm_status mpm_get_grid(mpm_ctx c, int32_t t, float* m, float* vbar) {
  if (!c) return MPM_ERR_INVALID_ARG;
  if (!c->has_state || t < 0 || t >= c->tape_len) return fail(c, MPM_ERR_CALL_ORDER, "step not on the tape");
  cudaSetDevice(c->cfg.device);
  const KParams& P = c->P;
  size_t nn = 1;
  for (int a = 0; a < c->D; ++a) nn *= P.res;
  nn *= P.B;
  float *dm = nullptr, *dv = nullptr;
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
  cudaFree(dm);
  cudaFree(dv);
  return s;
}

mpm_status mpm_get_step_info(mpm_ctx c, int32_t t, int32_t out[3]) {
  if (!c || !out) return MPM_ERR_INVALID_ARG;
  if (!c->has_state || t < 0 || t >= c->tape_len) return fail(c, MPM_ERR_CALL_ORDER, "step not on the tape");
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

mpm_status mpm_add_seed(mpm_ctx c, int32_t t, const float* dLdx, const float* dLdv, const float* dLdF,
                        const float* dLdC) {
  if (!c || t < 0 || t > c->cfg.max_steps) return MPM_ERR_INVALID_ARG;
  cudaSetDevice(c->cfg.device);
  const size_t NT = c->P.NT, D = c->D;
  const size_t n = NT * (2 * D + 2 * D * D);
  float*& b = c->seeds[t];
  if (!b) {
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
  for (auto& kv : c->seeds) cudaFree(kv.second);
  c->seeds.clear();
  return MPM_OK;
}

mpm_status mpm_enable_mass_grad(mpm_ctx c, int32_t on) {
  if (!c) return MPM_ERR_INVALID_ARG;
  c->mass_grad = on != 0;
  c->mass_grad_valid = false;
  return MPM_OK;
}

mpm_status mpm_grad_mass(mpm_ctx c, float* dmass) {
  if (!c || !dmass) return MPM_ERR_INVALID_ARG;
  if (!c->has_grad || !c->mass_grad_valid)
    return fail(c, MPM_ERR_CALL_ORDER, "mpm_grad_mass needs mpm_enable_mass_grad(1) before mpm_backward");
  cudaSetDevice(c->cfg.device);
  CK(cudaMemcpyAsync(dmass, c->dmass, (size_t)c->P.NT * sizeof(float), cudaMemcpyDefault, c->stream));
  return sync_and_check(c, "grad_mass");
}

}  // extern "C"
