/*
 * mpm.h -- C ABI of the B200-native differentiable MLS-MPM step
 *          (ChainQueen, arXiv 1810.01054; library paper_1810_01054_b200/libmpm.so, sm_100a).
 *
 * The problem statement follows the paper: a "memo" holds a whole rollout plus the initial
 * state p0 and the parameters used at every step (Fig. 2 caption P:173); the
 * caller asks for the gradient of a loss on the final state with respect to the initial
 * state and to the parameters, here the per-step actuation and the
 * per-particle Young's modulus / Poisson ratio.
 *
 *   forward  = P2G (Eqs. 3-5, with S1 P:430) -> grid (Eq. 6, plus
 *              gravity and wall friction) -> G2P (Eqs. 7-10);
 *   backward = the supplement's steps A-L per step, chained from the last step
 *              to the first.
 * Readings of the paper where it is silent are DESIGN.md R1-R19 (neo-Hookean psi, quadratic
 * B-spline, wall bands, epsilon, ...).
 *
 * Conventions
 *  - Ownership: the context owns every device buffer it allocates.  Input pointers are
 *    borrowed for the duration of the call and copied; they may be host (pageable or pinned)
 *    or device pointers (UVA, detected by the CUDA runtime).  Output buffers belong to the
 *    caller and may also be host or device.
 *  - Layout of user arrays (row-major, fp32 unless stated):
 *      x, v          [batch][n_particles][dim]
 *      F, C          [batch][n_particles][dim][dim]   (F[p][row][col])
 *      mass, vol, E, nu            [batch][n_particles]
 *      actuator_id   [batch][n_particles] int32, -1 = not actuated, else in [0, n_actuators)
 *      actuation a   [batch][max_steps][n_actuators][dim]   (sigma_pa = act_strength*Diag(a))
 *    All user-visible arrays are in the user's particle order; the per-step sort is internal.
 *  - Errors: status codes only; nothing throws across the ABI.  Device-side faults (particle
 *    outside the domain, inverted element) are latched on the device as (code, step,
 *    particle) and returned by the synchronising call that ends mpm_forward / mpm_backward.
 *    After MPM_ERR_OUT_OF_DOMAIN / MPM_ERR_INVERTED the context refuses forward/backward
 *    until mpm_set_state.  mpm_last_error() returns a human-readable message.
 *  - Streams: all work is ordered on config.stream (a cudaStream_t; NULL = the legacy
 *    default stream).  mpm_forward, mpm_backward, mpm_get_*, mpm_grad synchronise the stream
 *    before returning.  One context per host thread.
 */
#ifndef MPM_H
#define MPM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mpm_ctx_s* mpm_ctx;

typedef enum {
  MPM_OK = 0,
  MPM_ERR_INVALID_ARG = 1,
  MPM_ERR_OOM = 2,
  MPM_ERR_CUDA = 3,
  MPM_ERR_OUT_OF_DOMAIN = 4, /* base index outside [0, res-3] (DESIGN R14)          */
  MPM_ERR_INVERTED = 5,      /* det F <= 0, ln J undefined (DESIGN R14)             */
  MPM_ERR_TAPE_FULL = 6,     /* forward beyond max_steps, or grid-slot arena full    */
  MPM_ERR_CALL_ORDER = 7,    /* e.g. backward before forward, grad before backward   */
  MPM_ERR_COMM = 8,          /* NCCL failure (slab mode)                             */
  MPM_ERR_OUT_OF_SLAB = 9,   /* particle left its slab's halo (slab mode, see below) */
  MPM_ERR_CFL = 10,          /* fuse_g2p2g: a particle moved too far in one step for the
                                dilated grid of the next step (needs |v| dt < dx)          */
  MPM_ERR_MIGRATE = 11       /* migrating slab mode: more leavers per side and step than
                                mig_cap, more particles than the storage capacity, or a
                                particle that crossed a whole slab in one step              */
} mpm_status;

typedef struct {
  int32_t dim;          /* 2 or 3                                                     */
  int32_t res;          /* grid nodes per axis, power of two, 16..4096; dx = 1/res     */
  int32_t batch;        /* B independent rollouts ...                                 */
  int32_t n_particles;  /* ... of N particles each (N < 2^25)                         */
  int32_t max_steps;    /* tape capacity T (the memo holds states 0..T)               */
  int32_t n_actuators;  /* K (0..64)                                                  */
  float dt;             /* time step                                                  */
  float gravity[3];     /* added on the grid after Eq. 6 (R5)                         */
  int32_t bound;        /* wall band width in nodes (R6), >= 0, 2*bound < res          */
  float friction[6];    /* c per wall (-x,+x,-y,+y,-z,+z); c < 0 => sticky (R6)        */
  float act_strength;   /* s in sigma_pa = s * Diag(a[t][k])  (R4)                    */
  int32_t device;       /* CUDA device ordinal                                        */
  void* stream;         /* cudaStream_t or NULL                                       */
  int32_t grid_slots;   /* grid-block slots per step in the tape arena; 0 = automatic: sized at
                           every mpm_set_state (twice the touched blocks of the state) and
                           doubled by mpm_forward when a spreading body overflows it (the steps
                           on the tape are kept and the forward resumes from the overflowing
                           step); with grid_slots > 0 an overflow is MPM_ERR_TAPE_FULL         */
  int32_t checkpoint_every; /* NEXT N2: 0 = the memo keeps every step (max_steps of tape);
                           k > 0 = the tape keeps one k-step segment and full states every
                           k steps (max_steps/k + 1 checkpoints); mpm_backward recomputes
                           each earlier segment from its checkpoint (one extra forward),
                           mpm_get_state / mpm_rewind of an evicted step recompute it      */
  int32_t material;     /* NEXT N3 constitutive model: 0 = neo-Hookean (R1),
                           1 = fixed-corotated, psi = mu |F - R|^2 + lam/2 (J - 1)^2 (R21)   */
  int32_t fuse_g2p2g;   /* NEXT N2: 1 = fused forward, one particle pass per
                           step: the G2P of step t also scatters step t+1's P2G into a
                           grid allocated as the one-block dilation of step t's occupied
                           blocks (results equal the unfused path up to fp32 summation
                           order).  Requires |v| dt < dx (else MPM_ERR_CFL).  A slab with
                           neighbours sums the windows of grid t+1 between two fused launches;
                           ignored in the migrating slab mode (arrivals join state t+1 after
                           its G2P) and with a controller (N1 needs state t+1 before step
                           t+1's P2G).  Group calls need the same value in every context.
                           0 = P2G and G2P as separate passes.                           */
} mpm_config;

/* Create a context on config->device.  Validates the config (MPM_ERR_INVALID_ARG) and
 * allocates the fixed-size buffers (MPM_ERR_OOM); the tape is allocated by mpm_set_state. */
mpm_status mpm_create(const mpm_config* config, mpm_ctx* out);
void mpm_destroy(mpm_ctx ctx);

/* Initial state p0 and constant per-particle parameters; resets the tape to t = 0,
 * clears every gradient and the error latch.  E > 0, 0 <= nu < 0.5, mass > 0, vol > 0. */
mpm_status mpm_set_state(mpm_ctx ctx, const float* x, const float* v, const float* F,
                         const float* C, const float* mass, const float* vol, const float* E,
                         const float* nu, const int32_t* actuator_id);

/* Open-loop actuation for every step, [batch][max_steps][n_actuators][dim]. */
mpm_status mpm_set_actuation(mpm_ctx ctx, const float* a);

/* Advance n_steps steps from the current tape end, appending states to the memo.
 * MPM_ERR_TAPE_FULL if the tape would exceed max_steps.                                 */
mpm_status mpm_forward(mpm_ctx ctx, int32_t n_steps);

/* Number of steps currently on the tape. */
int32_t mpm_tape_length(mpm_ctx ctx);

/* Truncate the tape to its first t steps (0 <= t <= tape length), keeping states 0..t, so
 * the rollout can be re-run from state t (e.g. with new actuation) without re-uploading.
 * Clears the error latch and the gradients.                                               */
mpm_status mpm_rewind(mpm_ctx ctx, int32_t t);

/* State at tape step t (0 <= t <= tape length), user particle order.  NULL = skip.
 * With checkpoint_every > 0 a step outside the resident segment is recomputed from the
 * nearest checkpoint (and becomes resident).  In slab mode with a communicator that
 * recompute exchanges windows, so the call is then collective over the ranks (as are
 * mpm_forward, mpm_rewind and mpm_backward).                                              */
mpm_status mpm_get_state(mpm_ctx ctx, int32_t t, float* x, float* v, float* F, float* C);

/* Reverse mode over the whole tape: seed dL/dstate at t = tape length, user order,
 * same layouts as x, v, F, C; NULL = zero.  Requires a forward tape (MPM_ERR_CALL_ORDER). */
mpm_status mpm_backward(mpm_ctx ctx, const float* dLdx, const float* dLdv, const float* dLdF,
                        const float* dLdC);

/* Gradients from the last mpm_backward: w.r.t. the initial state (user order), E and nu
 * [batch][n], and the actuation [batch][max_steps][n_actuators][dim] (steps beyond the tape
 * length are 0).  NULL = skip.  MPM_ERR_CALL_ORDER before any backward.                 */
mpm_status mpm_grad(mpm_ctx ctx, float* dx0, float* dv0, float* dF0, float* dC0, float* dE,
                    float* dnu, float* da);

/* NEXT N3: dL/dm_p [batch][n] (user order) from the last mpm_backward -- the gradient behind
 * the paper's physical-parameter inference (density of a ball).  Derived by the chain
 * rule through Eqs. 3-5 (m enters m_i, m v and the m C part of G).          */
mpm_status mpm_grad_mass(mpm_ctx ctx, float* dmass);
/* Opt-in switch for the mass gradient (off by default: it costs ~15% of the P2G^T kernel).
 * mpm_grad_mass returns MPM_ERR_CALL_ORDER unless the last backward ran with it on.      */
mpm_status mpm_enable_mass_grad(mpm_ctx ctx, int32_t on);

/* NEXT N4: register an additive seed dL/dstate_t for state t (0 <= t <= max_steps), user
 * order, layouts as mpm_get_state; NULL = 0.  mpm_backward then differentiates the running
 * loss sum_t L_t(state_t) (P:348-349 goal-velocity reward, P:363 costs): the adjoint of
 * state t gets the seed added before step t-1 is reversed; the seed at t = tape length is
 * added to mpm_backward's own.  Seeds persist until mpm_clear_seeds; each costs
 * (2d + 2d^2) * batch * n floats of device memory (MPM_ERR_OOM if that fails).           */
mpm_status mpm_add_seed(mpm_ctx ctx, int32_t t, const float* dLdx, const float* dLdv,
                        const float* dLdF, const float* dLdC);
mpm_status mpm_clear_seeds(mpm_ctx ctx);

/* Message of the last failed call on ctx; with ctx = NULL, why the calling thread's last
 * mpm_create failed (invalid config field, cudaSetDevice, OOM size), or "null context".   */
const char* mpm_last_error(mpm_ctx ctx);

/* ---- NEXT N1: closed-loop controller embedded in P2G (Fig. 2 caption P:84) ----
 * With a controller set, every forward step t first computes, per rollout,
 *   z_t = [target (d), CoM_k (d) for k < K, V_k (d) for k < K]   (length nz = d (1 + 2K)),
 *   CoM_k / V_k = mass-weighted mean position / velocity of the particles with actuator_id k
 *   (the "composed soft components" of P:279, DESIGN R20), and
 *   a_t = tanh(W z_t + b)  -> the actuation of step t ([K][d], sigma_pa = s Diag(a), R4),
 * overwriting that step of the mpm_set_actuation buffer.  mpm_backward then adds the
 * controller's closed-loop terms to dL/dx_p, dL/dv_p of every state and accumulates
 * dL/dW, dL/db, dL/dtarget (summed over steps and rollouts), read by mpm_grad_controller.
 * W: [K*d][nz] row-major, b: [K*d], target: [d]; host or device pointers, copied.
 * Needs mpm_set_state first (group masses), n_actuators >= 1, every group non-empty in
 * every rollout (MPM_ERR_INVALID_ARG), no slab neighbours.  W = NULL switches it off.      */
mpm_status mpm_set_controller(mpm_ctx ctx, const float* W, const float* b, const float* target);
mpm_status mpm_grad_controller(mpm_ctx ctx, float* dW, float* db, float* dtarget);

/* ---- slab mode: one large rollout sharded by x-slab (configs[4] "8M particles
 * slab-sharded") ----
 * A context simulates the particles of one x-slab [x_lo, x_hi) of node planes (ownership
 * by base_x at t = 0, fixed for the rollout).  Nodes that two slabs can both touch lie in a
 * window of 2*halo_blocks block-planes (block = 4 nodes in 3D, 8 in 2D) centred on each
 * slab boundary; the exchange is the symmetric sum of those windows after P2G (Eq. 3-5 are
 * sums over ALL particles) and after G2P^T (the adjoint of that sum), so every node a rank
 * reads holds the whole-body value.  A particle may drift at most halo_blocks*block - 2
 * nodes past the slab (base_x in [x_lo - h, x_hi + h - 3], h = halo_blocks*block, on a side
 * that has a neighbour); beyond that forward latches MPM_ERR_OUT_OF_SLAB.  The actuation is
 * shared: after mpm_backward / mpm_group_backward, mpm_grad's da is summed over all slabs.
 *
 * mpm_set_slab: before mpm_set_state; batch must be 1; x_lo, x_hi multiples of the block
 *   size, 0 <= x_lo < x_hi <= res; a side with a neighbour (x_lo > 0, x_hi < res) needs
 *   x_hi - x_lo >= 2h and its window inside the domain.  Allocates 4 window buffers of
 *   2*halo_blocks*(res/block)^(dim-1)*64 float4 each.
 * mpm_comm_unique_id / mpm_comm_init: one context per GPU, one process per GPU; rank r's
 *   left neighbour is rank r-1 (ranks ordered by slab).  The exchange is a grouped NCCL
 *   send/recv with the two neighbours on config.stream; the da sum an NCCL all-reduce.
 *   mpm_comm_init is collective over the world (blocks until all ranks call it).
 *   libnccl.so.2 is loaded at the first NCCL call: one already in the process if any, else the
 *   file named by the environment variable MPM_NCCL_LIB (the Python binding sets it to the
 *   NCCL that torch bundles), else the loader's search path; none -> MPM_ERR_COMM.
 * mpm_group_forward / mpm_group_backward: the same exchange between n contexts of ONE
 *   process (adjacent slabs in x order, one device, one stream), done as device-to-device
 *   copies between the phases of every step -- a single-GPU emulation of the sharded run
 *   used by the parity tests; no kernel waits on another.  Seeds: arrays of n pointers
 *   (user order of each context) or NULL.                                                 */
mpm_status mpm_set_slab(mpm_ctx ctx, int32_t x_lo, int32_t x_hi, int32_t halo_blocks);

/* ---- migrating slab mode ("halo exchange of ghost grid nodes and migrating
 * particles") ----
 * As mpm_set_slab, but ownership is Eulerian: at EVERY step a particle belongs to the slab
 * whose [x_lo, x_hi) holds its base_x (the first slab also takes base_x < x_lo, the last
 * base_x >= x_hi), so a body may travel across any number of slab boundaries (no drift bound).
 * After the G2P of each step the particles whose base_x left the slab are packed (state + user
 * index) and exchanged with the x-neighbour (one grouped exchange per step; fixed-size buffers
 * of mig_cap records per side), and the arrivals are appended to the next state.  The window
 * sums of mpm_set_slab stay.  The send / receive buffers of every step stay on the tape: the
 * backward returns the adjoint of every arrival to the rank it came from and fills the slots of
 * the particles that left with the adjoints coming back (reverse migration), so each rank's
 * reverse pass sees exactly the particles it simulated at that step.
 *   - config.n_particles is this context's STORAGE capacity (live particles at any step;
 *     MPM_ERR_MIGRATE beyond it); n_global is the whole body's particle count: every array in
 *     user order (mpm_set_state, mpm_get_state, seeds, mpm_grad, mpm_grad_mass) spans the whole
 *     body, [n_global] leading.  mpm_set_state keeps the particles the slab owns at t = 0.
 *     mpm_get_state(t) and mpm_grad's dx0, dv0, dF0, dC0 write this slab's particles (owned at
 *     t, resp. at 0) and zeros elsewhere: the sum over the slabs is the whole body.  dE, dnu,
 *     dmass and da are the whole-body gradients on every slab (summed over the slabs by the
 *     backward: NCCL all-reduce, or in-process for mpm_group_backward).
 *   - mig_cap: records per side and step (0 = max(1024, capacity / 64)).
 *   - batch 1; checkpoint_every 0; no controller; no CUDA graphs; fuse_g2p2g is ignored.
 *   - mpm_group_forward / mpm_group_backward drive adjacent migrating contexts of one process
 *     (the same kernels, device copies in place of the exchanges).                           */
mpm_status mpm_set_slab_migrating(mpm_ctx ctx, int32_t x_lo, int32_t x_hi, int32_t halo_blocks,
                                  int32_t n_global, int32_t mig_cap);

/* Host-staged transport for the slab exchanges (an alternative to mpm_comm_init's NCCL, e.g.
 * gloo through torch.distributed for multi-process tests where the ranks share a GPU or have
 * none for NCCL): at every exchange the library synchronises its stream, copies the send
 * buffers to pinned host memory and calls fn(user, kind, send_left, send_right, recv_left,
 * recv_right, bytes) with host pointers (NULL on a side without a neighbour); fn must send
 * send_left to the left neighbour's recv_right (and send_right to the right neighbour's
 * recv_left), fill recv_left / recv_right, and return 0.  kind: MPM_XCHG_WINDOW (grid windows),
 * MPM_XCHG_MIGRATE (migrant records), MPM_XCHG_MIGRATE_ADJ (their adjoints, backward),
 * MPM_XCHG_REDUCE (fn must overwrite send_left with the elementwise sum over all ranks; the
 * right pointers are NULL: the da / dmu / dlam / dmass sums of the backward).  With a transport
 * set, forward/backward/get_state are collective over the ranks as with NCCL.  fn = NULL unsets. */
enum { MPM_XCHG_WINDOW = 0, MPM_XCHG_MIGRATE = 1, MPM_XCHG_MIGRATE_ADJ = 2, MPM_XCHG_REDUCE = 3 };
typedef int (*mpm_transport_fn)(void* user, int32_t kind, const float* send_left, const float* send_right,
                                float* recv_left, float* recv_right, size_t bytes);
mpm_status mpm_set_transport(mpm_ctx ctx, mpm_transport_fn fn, void* user);
mpm_status mpm_comm_unique_id(char out[128]);
mpm_status mpm_comm_init(mpm_ctx ctx, int32_t rank, int32_t world, const char id[128]);
mpm_status mpm_group_forward(mpm_ctx* ctxs, int32_t n_ctx, int32_t n_steps);
mpm_status mpm_group_backward(mpm_ctx* ctxs, int32_t n_ctx, const float* const* dLdx,
                              const float* const* dLdv, const float* const* dLdF,
                              const float* const* dLdC);

/* ---- introspection, used by the parity tests (all synchronous) ---- */

/* (Introspection calls need step t resident: with checkpoint_every > 0, inside the current
 * segment; otherwise MPM_ERR_CALL_ORDER.)
 * Binning of tape step t (north_star item 1): positions as stored for step t in the
 * internal storage order (x_store [B*N][dim]), the storage-to-user map orig [B*N], the
 * keys [B*N] computed from x_store, the stable sort perm [B*N] (sorted slot -> storage
 * index) and block_start [B*nb + 1], nb = (res/Bb)^dim, Bb = 4 (3D) / 8 (2D).  t < tape
 * length.  NULL = skip.                                                                  */
mpm_status mpm_get_binning(mpm_ctx ctx, int32_t t, float* x_store, int32_t* orig,
                           int32_t* key, int32_t* perm, int32_t* block_start);

/* Grid of tape step t as stored in the memo, dense [B][res^dim]: node mass m and vbar =
 * p/m + dt g (before the wall projection, R5/R6); 0 on untouched nodes.                 */
mpm_status mpm_get_grid(mpm_ctx ctx, int32_t t, float* m, float* vbar);

/* Block table of tape step t: out[0] = occupied grid blocks, out[1] = touched blocks (grid
 * slots, 64 nodes each), out[2] = first arena slot of the step.  t < tape length.        */
mpm_status mpm_get_step_info(mpm_ctx ctx, int32_t t, int32_t out[3]);

/* Per-kernel device time (ms) and launch counts accumulated while profiling is on; names
 * are returned as a ';'-separated list.  n_kernels in/out. */
mpm_status mpm_set_profiling(mpm_ctx ctx, int32_t on);
mpm_status mpm_get_profile(mpm_ctx ctx, int32_t* n_kernels, float* ms, int64_t* launches,
                           char* names, int32_t names_len);
/* Total kernel launches issued by this context since creation (a replayed graph counts the
 * kernels it launches). */
int64_t mpm_launch_count(mpm_ctx ctx);

/* CUDA graphs for the step loops (off by default).  With on != 0, the launches of an
 * mpm_forward(n) call -- and of the backward's loop over the memo's steps -- are captured
 * into a CUDA graph the first time a (direction, start step, step count) occurs and replayed
 * on later calls with the same triple (the launch-bound small configurations: P:167 and
 * P:218 put the paper's TF overheads on per-op launches).  The graph computes exactly what
 * the launches do: same kernels, same arguments, same stream order.  Loops that cannot be
 * captured run as plain launches: n < 2 steps, checkpoint_every > 0 (recompute segments
 * synchronise), slab neighbours (NCCL), profiling on.  Graphs are dropped when a call changes
 * what the loops launch (mpm_set_controller, a new mpm_add_seed step, mpm_clear_seeds,
 * mpm_enable_mass_grad) and on mpm_set_graphs(ctx, 0) / mpm_destroy; at most 16 executables
 * are kept (least recently used dropped first).
 * Errors: MPM_ERR_INVALID_ARG if config.stream is NULL (the legacy stream cannot be captured).
 * A capture or instantiation failure returns MPM_ERR_CUDA and poisons the context (its host
 * bookkeeping advanced for launches that never ran): call mpm_set_state before the next step. */
mpm_status mpm_set_graphs(mpm_ctx ctx, int32_t on);

#ifdef __cplusplus
}
#endif
#endif /* MPM_H */
