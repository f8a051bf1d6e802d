// mpm_kernels.cuh -- sm_100a kernels of the differentiable MLS-MPM step
// (ChainQueen, arXiv 1810.01054).  Product code: shares nothing with oracle/.
//
// Citations: P:<line> = PAPER.md line; R<k> = DESIGN.md reading k.
//
// Layout:
//   particle state, tape step t: AoSoA, "storage order t" -- groups of 32 particles, component-
//   major inside a group (rix below; MPM_AOSOA=0: plain SoA, comp * NT + j)
//       comp(x_a) = a, comp(v_a) = D + a, comp(C_ab) = 2D + aD + b, comp(F_ab) = 2D + D^2 + aD + b
//     storage order t+1 == the sorted (block, cell, index) order of step t.
//   grid: sparse, one 64-node slot (1 KiB, float4 per node) per touched block of Bb^D
//     nodes (Bb = 4 in 3D, 8 in 2D); node float4 = (p_x, p_y, p_z, m) after P2G,
//     (vbar_x, vbar_y, vbar_z, m) after the grid update; slots of step t live in the tape arena.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// occupancy targets (min CTAs per SM) of the block kernels; tuned on B200
#ifndef MPM_G2P_MINB
#define MPM_G2P_MINB 4
#endif
#ifndef MPM_P2GT_MINB
#define MPM_P2GT_MINB 4
#endif
#ifndef MPM_P2GT_PF
#define MPM_P2GT_PF 0  // block-prologue L2 prefetch of the records: measured 12 us slower (the loads overlap anyway)
#endif
#ifndef MPM_G2P_PF
#define MPM_G2P_PF 1
#endif
#ifndef MPM_FFMA2
#define MPM_FFMA2 1  // packed fp32x2 FMAs (sm_100 FFMA2) in the stencil sums
#endif
#ifndef MPM_FUSE_STAGE_FIRST
#define MPM_FUSE_STAGE_FIRST 1
#endif
#ifndef MPM_FUSE_CAP
#define MPM_FUSE_CAP 512
#endif
#ifndef MPM_FUSE_FX
#define MPM_FUSE_FX 1
#endif
#ifndef MPM_FUSE_MINB
#define MPM_FUSE_MINB (MPM_FUSE_FX ? 4 : 3)
#endif
#ifndef MPM_SCAT_PF
#define MPM_SCAT_PF 1
#endif
#ifndef MPM_FFMA2_SCAT
#define MPM_FFMA2_SCAT 1
#endif
#ifndef MPM_FFMA2_P2GT
#define MPM_FFMA2_P2GT 3  // packed FFMA2 in both P2G^T passes: -6.9 us once the park freed registers (round 1: +3 us at the register cliff)
#endif
#ifndef MPM_P2GT_THREADS
#define MPM_P2GT_THREADS 128
#endif
#ifndef MPM_P2GT_SIG_EARLY
#define MPM_P2GT_SIG_EARLY 1  // the actuation load issued before the v-pass: measured -2 us (P2G^T 136.0 -> 134.0)
#endif
#ifndef MPM_P2GT_PARK
#define MPM_P2GT_PARK 3  // record rows parked in shared memory (1: dL/dx, dL/dF; 2: + H; 3: + v, C): -9.5 us
#endif
#ifndef MPM_GRIDT_FUSED
#define MPM_GRIDT_FUSED 1  // gridT folded into P2G^T's tile staging (no k_grid_adj launch): 1 = small
                           // problems (the SPLIT path), 2 = always (C4: P2G^T +9 us, bench +8 us)
#endif
#ifndef MPM_P2GT_IDXSM
#define MPM_P2GT_IDXSM 1  // P2G^T: each item's perm / orig staged in shared memory with the tile (-0.8 us)
#endif
#ifndef MPM_FUSE_SPERM
#define MPM_FUSE_SPERM 1  // fused G2P2G: the in-block sort's order kept in shared memory for the producer (-0.5 us)
#endif
#ifndef MPM_P2GT_CLAIM
#define MPM_P2GT_CLAIM 1  // P2G^T work items claimed and decoded by thread 0 (claim_item)
#endif

#ifndef MPM_SCAT_FX
#define MPM_SCAT_FX 1
#endif
#ifndef MPM_SCAT_MINB
#define MPM_SCAT_MINB (MPM_SCAT_FX ? 4 : 3)
#endif
#ifndef MPM_SCATA_FX
#define MPM_SCATA_FX 1
#endif
#ifndef MPM_SCATA_MINB
#define MPM_SCATA_MINB (MPM_SCATA_FX ? 4 : 3)
#endif

namespace mpm {

constexpr int kCPB = 64;         // cells (and nodes) per grid block
constexpr int kThreads = 256;    // CTA size of the block-tile kernels
constexpr int kCap = 512;        // particles per producer chunk
constexpr int kSortCap = 2048;   // in-smem cell sort capacity (larger blocks use scratch)
#ifndef MPM_SCAN_THREADS
#define MPM_SCAN_THREADS 512  // 512-block tiles: C4 scan -1.4 us (256: 14.4, 1024: 12.7 but C3 +2 us)
#endif
constexpr int kScanTile = MPM_SCAN_THREADS;  // grid blocks per scan tile = threads of a scan CTA
#ifndef MPM_SCAT_CTAS
#define MPM_SCAT_CTAS 8  // k_scatter CTAs per SM (256 threads)
#endif
#ifndef MPM_GRIDT_CTAS
#define MPM_GRIDT_CTAS 8  // k_grid_adj CTAs per SM (256 threads)
#endif
#ifndef MPM_SCATQ
#define MPM_SCATQ 4
#endif
constexpr int kScatQ = MPM_SCATQ;  // particles per thread in k_scatter
constexpr int kCapPerm = 512;    // fused G2P2G: the block's sorted order kept in shared memory
constexpr int kIdxCap = 512;     // P2G^T: an item's perm / orig entries held in shared memory
constexpr int kMaxAct = 64;      // n_actuators cap (mpm_create validates)  // grid blocks per scan tile (one per thread)
constexpr float kEps = 1e-10f;   // step-L epsilon (R7)

// Programmatic dependent launch (sm_90+): a kernel of the step path waits for its
// predecessor's completion (and memory) before touching any of its outputs, then lets its own
// dependent start launching; with the PDL launch attribute the next kernel's launch and CTA
// placement overlap this kernel's tail.  No-ops for ordinary launches.
#define MPM_PDL_ENTRY()                                    \
  do {                                                     \
    asm volatile("griddepcontrol.wait;" ::: "memory");     \
    asm volatile("griddepcontrol.launch_dependents;" ::);  \
  } while (0)

// Debug builds (-DMPM_DEBUG_BOUNDS=1; tools/build_variant.sh): index checks on the shared-
// memory tiles, payload and sort buffers and the grid-slot arena; a violated check prints
// the site and traps.  Compiled out otherwise.
#ifndef MPM_DEBUG_BOUNDS
#define MPM_DEBUG_BOUNDS 0
#endif
#if MPM_DEBUG_BOUNDS
#define MPM_CHECK(cond)                                                                  \
  do {                                                                                   \
    if (!(cond)) {                                                                       \
      printf("MPM_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             blockIdx.x, threadIdx.x);                                                   \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)
#else
#define MPM_CHECK(cond) \
  do {                  \
  } while (0)
#endif

enum ErrCode { E_OK = 0, E_DOMAIN = 4, E_INVERTED = 5, E_TAPE_FULL = 6, E_SLAB = 9, E_FUSE = 10, E_MIGRATE = 11 };

template <int D> struct Dim;
template <> struct Dim<3> {
  static constexpr int BB = 4, LOG_BB = 2, NS = 27, TE = 6, TN = 216, S = 24;
};
template <> struct Dim<2> {
  static constexpr int BB = 8, LOG_BB = 3, NS = 9, TE = 10, TN = 100, S = 12;
};

// Step-invariant parameters, passed by value.
struct KParams {
  int res, B, N, NT, nbpa, nb, NBT, K, T;  // T = max_steps (actuation stride)
  float dt, dx, fres;                       // dx = 1/res, fres = res
  float g[3];
  int bound;
  float fric[6];
  float act_s;
  int slots_per_step;                       // per-step cap of touched blocks
  int arena_slots;                          // capacity of the tape grid arena
  int slab_lo, slab_hi;                     // allowed base_x range (inclusive); slab mode
  int material;                             // 0 = neo-Hookean (R1), 1 = fixed-corotated (R21)
  int nz;                                   // controller observation length d (1 + 2K) (NEXT N1)
};

// Migrating slab mode (separate from KParams so the step kernels' parameters are unchanged): a
// particle is owned by the slab whose [own_lo, own_hi) holds its base_x, at every step.
struct MigParams {
  int migrate;
  int own_lo, own_hi;
  int mig_cap;  // migrant records per side and step
};

// Per-step bookkeeping record, info[t * kInfo + field]
constexpr int kInfo = 12;
enum { I_NOCC = 0, I_NTOUCH = 1, I_BASE = 2, I_WORK = 3, I_WORK2 = 4, I_OK = 5, I_WORK3 = 6, I_WORK4 = 7,
       I_NSLOT = 8,    // storage slots of state t (migrating slab mode; live + left-behind holes)
       I_NBIG = 9 };   // occupied blocks with >= kBigBlock particles: occ_list[0, I_NBIG); the others
                       // fill occ_list from its end (occ_list[NBT - 1 - i], i < I_NOCC - I_NBIG)
constexpr int kBigBlock = 256;  // particles: the "long" work items claimed first (k_scan_lookback)

// Migrating slab mode: a particle whose base_x leaves the slab after G2P gets this key (it is
// not binned, gathered or scattered on this rank at the next step -- a hole in the storage)
constexpr int kDeadKey = -2;
// migrant record in a send / receive buffer: the new state (S floats, H = F - I), the user index
// and the sender's storage slot (bit-cast into floats); buffer = int count (padded to 4 floats)
// followed by mig_cap records
template <int D> struct Mig { static constexpr int S = Dim<D>::S, U = S, K = S + 1, R = S + 2, HDR = 4; };

struct ErrLatch { int code, step, particle, pad; };

__device__ __forceinline__ void latch(ErrLatch* e, int code, int step, int particle) {
  if (atomicCAS(&e->code, 0, code) == 0) {
    e->step = step;
    e->particle = particle;
  }
}

// ------------------------------------------------------------------------------------
// index helpers
// ------------------------------------------------------------------------------------
// Particle records (states on the tape, adjoints): component comp of particle j.  AoSoA: a
// particle's 32-lane group holds its S components as 32-float rows, so after the per-particle
// group base every component is an immediate offset (the SoA form needs a 64-bit comp * NT
// multiply-add per access); warps reading 32 consecutive particles stay fully coalesced.
#ifndef MPM_AOSOA
#define MPM_AOSOA 1
#endif
__host__ __device__ __forceinline__ size_t rixs(int S, int comp, int j, size_t NT) {
#if MPM_AOSOA
  (void)NT;
  return ((size_t)(j >> 5) * S + comp) * 32 + (j & 31);
#else
  return (size_t)comp * NT + j;
#endif
}
// floats of a record buffer of NT particles (AoSoA pads to a whole group)
__host__ __device__ __forceinline__ size_t rec_floats(int S, size_t NT) {
#if MPM_AOSOA
  return (size_t)S * ((NT + 31) / 32 * 32);
#else
  return (size_t)S * NT;
#endif
}

template <int D> __device__ __forceinline__ int comp_x(int a) { return a; }
template <int D> __device__ __forceinline__ int comp_v(int a) { return D + a; }
template <int D> __device__ __forceinline__ int comp_C(int a, int b) { return 2 * D + a * D + b; }
template <int D> __device__ __forceinline__ int comp_F(int a, int b) { return 2 * D + D * D + a * D + b; }
template <int D> __device__ __forceinline__ size_t rix(int comp, int j, size_t NT) {
  return rixs(2 * D + 2 * D * D, comp, j, NT);
}

// block linear index inside one rollout from block coords (row-major, axis 0 slowest)
template <int D> __device__ __forceinline__ int block_lin(const int* b, int nbpa) {
  int l = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) l = l * nbpa + b[a];
  return l;
}
template <int D> __device__ __forceinline__ int cell_lin(const int* c) {
  int l = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) l = l * Dim<D>::BB + c[a];
  return l;
}

// ------------------------------------------------------------------------------------
// quadratic B-spline stencil (R2) in fp32.  xg = x * res is exact (res = 2^k); the base
// decision floor(xg - 0.5f) is the binning decision of R17.
// ------------------------------------------------------------------------------------
template <int D> struct Stencil {
  int base[D];
  float fx[D];
  float w[D][3];
};

__device__ __forceinline__ int base_of(float x, float fres) {
  float xg = x * fres;
  return (int)floorf(xg - 0.5f);
}

template <int D>
__device__ __forceinline__ void make_stencil(const float* x, float fres, Stencil<D>& s) {
#pragma unroll
  for (int a = 0; a < D; ++a) {
    float xg = x[a] * fres;
    int b = (int)floorf(xg - 0.5f);
    float f = xg - (float)b;  // in [0.5, 1.5), exact
    s.base[a] = b;
    s.fx[a] = f;
    float u0 = 1.5f - f, u1 = f - 1.0f, u2 = f - 0.5f;
    s.w[a][0] = 0.5f * u0 * u0;
    s.w[a][1] = 0.75f - u1 * u1;
    s.w[a][2] = 0.5f * u2 * u2;
  }
}

// dN/du at the three nodes, u = fx - o:  (fx - 1.5, -2 (fx - 1), fx - 0.5)
__device__ __forceinline__ void stencil_dw(float f, float* dw) {
  dw[0] = f - 1.5f;
  dw[1] = -2.0f * (f - 1.0f);
  dw[2] = f - 0.5f;
}

// ------------------------------------------------------------------------------------
// neo-Hookean Kirchhoff stress (R1) + actuation (S1, R3/R4):
//   tau = mu (F F^T - I) + lam ln J I + F Diag(sig) F^T   ( = P_total F^T )
// ------------------------------------------------------------------------------------
template <int D> __device__ __forceinline__ float det(const float (&F)[D][D]);
template <> __device__ __forceinline__ float det<2>(const float (&F)[2][2]) {
  return F[0][0] * F[1][1] - F[0][1] * F[1][0];
}
template <> __device__ __forceinline__ float det<3>(const float (&F)[3][3]) {
  return F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) -
         F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0]) +
         F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]);
}

// inverse transpose F^{-T}
template <int D> __device__ __forceinline__ void inv_T(const float (&F)[D][D], float J, float (&G)[D][D]);
template <> __device__ __forceinline__ void inv_T<2>(const float (&F)[2][2], float J, float (&G)[2][2]) {
  float iJ = 1.0f / J;
  G[0][0] = F[1][1] * iJ; G[0][1] = -F[1][0] * iJ;
  G[1][0] = -F[0][1] * iJ; G[1][1] = F[0][0] * iJ;
}
template <> __device__ __forceinline__ void inv_T<3>(const float (&F)[3][3], float J, float (&G)[3][3]) {
  float iJ = 1.0f / J;
  // cofactor matrix / J = F^{-T}
  G[0][0] = (F[1][1] * F[2][2] - F[1][2] * F[2][1]) * iJ;
  G[0][1] = (F[1][2] * F[2][0] - F[1][0] * F[2][2]) * iJ;
  G[0][2] = (F[1][0] * F[2][1] - F[1][1] * F[2][0]) * iJ;
  G[1][0] = (F[0][2] * F[2][1] - F[0][1] * F[2][2]) * iJ;
  G[1][1] = (F[0][0] * F[2][2] - F[0][2] * F[2][0]) * iJ;
  G[1][2] = (F[0][1] * F[2][0] - F[0][0] * F[2][1]) * iJ;
  G[2][0] = (F[0][1] * F[1][2] - F[0][2] * F[1][1]) * iJ;
  G[2][1] = (F[0][2] * F[1][0] - F[0][0] * F[1][2]) * iJ;
  G[2][2] = (F[0][0] * F[1][1] - F[0][1] * F[1][0]) * iJ;
}

template <int D>
__device__ __forceinline__ void kirchhoff(const float (&F)[D][D], float mu, float lam,
                                          const float* sig, float (&tau)[D][D], float lnJ) {
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = a; b < D; ++b) {
      float ff = 0.f, fsf = 0.f;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        ff = fmaf(F[a][c], F[b][c], ff);
        fsf = fmaf(F[a][c] * sig[c], F[b][c], fsf);
      }
      float t = mu * (ff - (a == b ? 1.f : 0.f)) + fsf;
      if (a == b) t += lam * lnJ;
      tau[a][b] = t;
      tau[b][a] = t;
    }
}

// The state stores the displacement gradient H = F - I instead of F (DESIGN.md 6,
// "numerics"): F is within ~1e-3 of I in these scenes, and fp32 F would carry an absolute
// rounding error that is large relative to the strain F - I the stress depends on.  With H,
// F F^T - I = H + H^T + H H^T and det F - 1 are formed without cancellation.
template <int D> __device__ __forceinline__ float det1m(const float (&H)[D][D]);  // det(I+H) - 1
template <> __device__ __forceinline__ float det1m<2>(const float (&H)[2][2]) {
  return H[0][0] + H[1][1] + (H[0][0] * H[1][1] - H[0][1] * H[1][0]);
}
template <> __device__ __forceinline__ float det1m<3>(const float (&H)[3][3]) {
  const float tr = H[0][0] + H[1][1] + H[2][2];
  const float m2 = (H[0][0] * H[1][1] - H[0][1] * H[1][0]) + (H[0][0] * H[2][2] - H[0][2] * H[2][0]) +
                   (H[1][1] * H[2][2] - H[1][2] * H[2][1]);
  return tr + m2 + det<3>(H);
}

template <int D>
__device__ __forceinline__ void load_H(const float* st, size_t NT, int j, float (&H)[D][D]) {
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) H[a][b] = __ldg(&st[rix<D>(comp_F<D>(a, b), j, NT)]);
}

template <int D>
__device__ __forceinline__ void F_of_H(const float (&H)[D][D], float (&F)[D][D]) {
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) F[a][b] = H[a][b] + (a == b ? 1.f : 0.f);
}

// F F^T - I from H
template <int D>
__device__ __forceinline__ float ffti(const float (&H)[D][D], int a, int b) {
  float acc = H[a][b] + H[b][a];
#pragma unroll
  for (int c = 0; c < D; ++c) acc = fmaf(H[a][c], H[b][c], acc);
  return acc;
}

// tau = mu (F F^T - I) + lam ln J I + F Diag(sig) F^T, from H (R1, S1)
template <int D>
__device__ __forceinline__ void kirchhoff_h(const float (&H)[D][D], float mu, float lam, const float* sig,
                                            float (&tau)[D][D], float lnJ) {
  float F[D][D];
  F_of_H<D>(H, F);
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = a; b < D; ++b) {
      float fsf = 0.f;
#pragma unroll
      for (int c = 0; c < D; ++c) fsf = fmaf(F[a][c] * sig[c], F[b][c], fsf);
      float t = fmaf(mu, ffti<D>(H, a, b), fsf);
      if (a == b) t = fmaf(lam, lnJ, t);
      tau[a][b] = t;
      tau[b][a] = t;
    }
}

// ------------------------------------------------------------------------------------
// Fixed-corotated material (NEXT N3, DESIGN R21), Kirchhoff form: with B = F F^T = V^2,
//   tau = 2 mu (B - V) + lam J (J - 1) I + F Diag(sig) F^T.
// E = B - I (exact from H) is diagonalised, E = Q diag(e) Q^T (cyclic Jacobi, fixed sweeps; robust
// for the near-degenerate E of small strains); V has eigenvalues s = sqrt(1 + e), and
// B - V = Q diag(e s / (s + 1)) Q^T carries no cancellation against I.
// ------------------------------------------------------------------------------------
template <int D> struct Stretch {
  float s[D];     // eigenvalues of V
  float g[D];     // eigenvalues of B - V
  float Q[D][D];  // eigenvectors (columns)
};

template <int P, int Q_, int D>
__device__ __forceinline__ void jacobi_rot(float (&A)[D][D], float (&Q)[D][D]) {
  const float apq = A[P][Q_];
  const float tau = A[Q_][Q_] - A[P][P];
  const float t = 2.f * apq * copysignf(1.f, tau) / (fabsf(tau) + sqrtf(fmaf(tau, tau, 4.f * apq * apq)) + 1e-30f);
  const float c = rsqrtf(fmaf(t, t, 1.f)), sn = t * c;
  A[P][P] -= t * apq;
  A[Q_][Q_] += t * apq;
  A[P][Q_] = A[Q_][P] = 0.f;
  if constexpr (D == 3) {
    constexpr int R = 3 - P - Q_;
    const float arp = A[R][P], arq = A[R][Q_];
    A[R][P] = A[P][R] = c * arp - sn * arq;
    A[R][Q_] = A[Q_][R] = sn * arp + c * arq;
  }
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const float qp = Q[k][P], qq = Q[k][Q_];
    Q[k][P] = c * qp - sn * qq;
    Q[k][Q_] = sn * qp + c * qq;
  }
}

template <int D>
__device__ __forceinline__ void left_stretch(const float (&H)[D][D], Stretch<D>& st) {
  float A[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      A[a][b] = ffti<D>(H, a, b);
      st.Q[a][b] = a == b ? 1.f : 0.f;
    }
  if constexpr (D == 2) {
    jacobi_rot<0, 1, 2>(A, st.Q);  // exact for 2x2
  } else {
#pragma unroll
    for (int sweep = 0; sweep < 5; ++sweep) {
      jacobi_rot<0, 1, 3>(A, st.Q);
      jacobi_rot<0, 2, 3>(A, st.Q);
      jacobi_rot<1, 2, 3>(A, st.Q);
    }
  }
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const float e = fmaxf(A[k][k], -0.999999f);
    const float sk = sqrtf(1.f + e);
    st.s[k] = sk;
    st.g[k] = e * sk / (sk + 1.f);
  }
}

// tau for the fixed-corotated model (R21, S1)
template <int D>
__device__ __forceinline__ void kirchhoff_fcr(const float (&H)[D][D], float mu, float lam, const float* sig,
                                              float (&tau)[D][D], float jm1) {
  Stretch<D> st;
  left_stretch<D>(H, st);
  float F[D][D];
  F_of_H<D>(H, F);
  const float lj = lam * (1.f + jm1) * jm1;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = a; b < D; ++b) {
      float fsf = 0.f, bv = 0.f;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        fsf = fmaf(F[a][c] * sig[c], F[b][c], fsf);
        bv = fmaf(st.Q[a][c] * st.g[c], st.Q[b][c], bv);
      }
      float t = fmaf(2.f * mu, bv, fsf);
      if (a == b) t += lj;
      tau[a][b] = t;
      tau[b][a] = t;
    }
}

// ------------------------------------------------------------------------------------
// Wall-band friction projection of step L (R6 band geometry, R7, R8), applied
// to a node's vbar on read.  Walls are axis aligned: n = +e_a (low wall), -e_a (high).
// ------------------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ bool in_band(const int* node, int res, int bound) {
  bool b = false;
#pragma unroll
  for (int a = 0; a < D; ++a) b |= (node[a] < bound) | (node[a] >= res - bound);
  return b;
}

// one wall: v <- proj(v), normal n = sgn * e_ax
template <int D>
__device__ __forceinline__ void project_wall(float* v, int ax, float sgn, float c) {
  if (c < 0.f) {
#pragma unroll
    for (int a = 0; a < D; ++a) v[a] = 0.f;
    return;
  }
  float ln = sgn * v[ax];
  if (ln >= 0.f) return;  // R8 identity branch
  float s2 = 0.f;
#pragma unroll
  for (int a = 0; a < D; ++a)
    if (a != ax) s2 = fmaf(v[a], v[a], s2);
  float lt = sqrtf(s2 + kEps);
  float lts = fmaxf(lt + c * ln, 0.f);
  float sc = lts / lt;
#pragma unroll
  for (int a = 0; a < D; ++a) v[a] = (a == ax) ? 0.f : v[a] * sc;
}

template <int D>
__device__ __forceinline__ void project_node(float* v, const int* node, const KParams& P) {
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (node[a] < P.bound) project_wall<D>(v, a, 1.f, P.fric[2 * a]);
    if (node[a] >= P.res - P.bound) project_wall<D>(v, a, -1.f, P.fric[2 * a + 1]);
  }
}

// adjoint of project_wall: g (= dL/dv*) -> dL/dv, given the wall's input v
template <int D>
__device__ __forceinline__ void project_wall_adj(const float* v, float* g, int ax, float sgn, float c) {
  if (c < 0.f) {
#pragma unroll
    for (int a = 0; a < D; ++a) g[a] = 0.f;
    return;
  }
  float ln = sgn * v[ax];
  if (ln >= 0.f) return;
  float s2 = 0.f;
#pragma unroll
  for (int a = 0; a < D; ++a)
    if (a != ax) s2 = fmaf(v[a], v[a], s2);
  float lt = sqrtf(s2 + kEps);
  float R = lt + c * ln;
  float H = (R >= 0.f) ? 1.f : 0.f;
  float lts = fmaxf(R, 0.f);
  float s = lts / lt;
  // v* = s * v_t ;  s = max(R,0)/lt ; ds/dlt = (H lt - lts)/lt^2 ; ds/dln = H c / lt
  float gs = 0.f;
#pragma unroll
  for (int a = 0; a < D; ++a)
    if (a != ax) gs = fmaf(g[a], v[a], gs);
  float k1 = gs * (H * lt - lts) / (lt * lt * lt);
  float gln = gs * H * c / lt;  // minus (g_vt . n) = 0 since v_t . n = 0 direction has g_vt_n = s g_n
  float gvt[D];
#pragma unroll
  for (int a = 0; a < D; ++a) gvt[a] = (a == ax) ? s * g[a] : fmaf(s, g[a], k1 * v[a]);
  // ln = sgn v_ax;  v_t = v - ln n  ->  dv = g_vt (I - n n^T) + (gln) n
#pragma unroll
  for (int a = 0; a < D; ++a) g[a] = (a == ax) ? sgn * gln : gvt[a];
}

// adjoint of project_node (reverse wall order, R6), g in/out, vbar = node input
template <int D>
__device__ __forceinline__ void project_node_adj(const float* vbar, float* g, const int* node,
                                                 const KParams& P) {
  // replay forward, storing the input of every active wall (at most 2 per axis, 1 in practice)
  float vin[2 * D][D];
  int wax[2 * D];
  float wsg[2 * D], wc[2 * D];
  int nw = 0;
  float v[D];
#pragma unroll
  for (int a = 0; a < D; ++a) v[a] = vbar[a];
#pragma unroll
  for (int a = 0; a < D; ++a) {
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      bool act = side == 0 ? (node[a] < P.bound) : (node[a] >= P.res - P.bound);
      if (act) {
#pragma unroll
        for (int q = 0; q < D; ++q) vin[nw][q] = v[q];
        wax[nw] = a;
        wsg[nw] = side == 0 ? 1.f : -1.f;
        wc[nw] = P.fric[2 * a + side];
        project_wall<D>(v, a, wsg[nw], wc[nw]);
        ++nw;
      }
    }
  }
  for (int w = nw - 1; w >= 0; --w) project_wall_adj<D>(vin[w], g, wax[w], wsg[w], wc[w]);
}

// ------------------------------------------------------------------------------------
// warp-aggregated histogram increment
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void warp_hist_add(int* cnt, int gb, bool valid) {
  unsigned vm = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  unsigned peers = __match_any_sync(vm, gb);
  int lane = threadIdx.x & 31;
  if (lane == __ffs(peers) - 1) atomicAdd(&cnt[gb], __popc(peers));
}

// key of a particle from its fp32 position (north_star item 1, R17); returns false when
// the base index is outside [0, res-3] (R14).
template <int D>
__device__ __forceinline__ int key_of(const float* x, int r, const KParams& P, int& gb, int& key) {
  int blk[D], cell[D];
  bool ok = true, in_slab = true;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    int b = base_of(x[a], P.fres);
    ok &= (b >= 0) & (b <= P.res - 3);
    if (a == 0) in_slab = (b >= P.slab_lo) & (b <= P.slab_hi);
    b = min(max(b, 0), P.res - 3);  // keep the bookkeeping in range; the error is latched
    blk[a] = b >> Dim<D>::LOG_BB;
    cell[a] = b & (Dim<D>::BB - 1);
  }
  gb = r * P.nb + block_lin<D>(blk, P.nbpa);
  key = gb * kCPB + cell_lin<D>(cell);
  return !ok ? E_DOMAIN : (!in_slab ? E_SLAB : E_OK);
}

// ------------------------------------------------------------------------------------
// set_state helpers
// ------------------------------------------------------------------------------------
// user AoS [N][D], [N][D][D] -> SoA state of n storage slots; slot j takes user particle
// idx[j] (migrating slab mode: this slab's members) or j; params -> {m, V, mu, lam}
template <int D>
__global__ void k_user_to_soa(KParams P, const float* __restrict__ x, const float* __restrict__ v,
                              const float* __restrict__ F, const float* __restrict__ C,
                              float* __restrict__ st, const int* __restrict__ idx, int n) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const size_t NT = P.NT;
  const size_t u = idx ? idx[j] : j;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    st[rix<D>(comp_x<D>(a), j, NT)] = x[u * D + a];
    st[rix<D>(comp_v<D>(a), j, NT)] = v ? v[u * D + a] : 0.f;
#pragma unroll
    for (int b = 0; b < D; ++b) {
      st[rix<D>(comp_C<D>(a, b), j, NT)] = C ? C[(u * D + a) * D + b] : 0.f;
      st[rix<D>(comp_F<D>(a, b), j, NT)] = F ? F[(u * D + a) * D + b] - (a == b ? 1.f : 0.f) : 0.f;  // H = F - I
    }
  }
}

__global__ void k_params(int NT, const float* __restrict__ m, const float* __restrict__ V,
                         const float* __restrict__ E, const float* __restrict__ nu,
                         float4* __restrict__ prm, int* __restrict__ bad) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= NT) return;
  float e = E[j], n = nu[j];
  // Lame parameters (R1)
  float mu = e / (2.f * (1.f + n));
  float lam = e * n / ((1.f + n) * (1.f - 2.f * n));
  if (!(m[j] > 0.f) || !(V[j] > 0.f) || !(e > 0.f) || !(n >= 0.f) || !(n < 0.5f)) atomicExch(bad, 1);
  prm[j] = make_float4(m[j], V[j], mu, lam);
}

// keys and block histogram of a stored state (storage slots [0, *nslot), or all NT); orig (if
// given) = identity, for t = 0 where storage order 0 = user order.  Migrating slab mode: a slot
// whose base_x is outside the slab (a particle that left at the previous step) is a hole.
template <int D>
__global__ void k_init_keys(KParams P, const float* __restrict__ st, int* __restrict__ key,
                            int* __restrict__ cnt, int* __restrict__ orig, ErrLatch* err,
                            const int* __restrict__ nslot, MigParams M) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  bool valid = j < (nslot ? *nslot : P.NT);
  int gb = 0, k = 0;
  if (valid) {
    float x[D];
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = st[rix<D>(comp_x<D>(a), j, P.NT)];
    if (M.migrate) {
      const int bx = base_of(x[0], P.fres);
      if (bx < M.own_lo || bx >= M.own_hi) {
        key[j] = kDeadKey;
        valid = false;
      }
    }
    if (valid) {
      if (const int e = key_of<D>(x, j / P.N, P, gb, k)) latch(err, e, 0, j);
      key[j] = k;
    }
    if (orig) orig[j] = j;
  }
  warp_hist_add(cnt, gb, valid);
}

// ------------------------------------------------------------------------------------
// block table of step t: exclusive scans of (count, occupied, touched) over all grid
// blocks, the occupied list, touched list and slot map.
// touched(b) = some block b - delta, delta in {0,1}^D, holds particles (a particle with
// base in block b' touches nodes of b' and b' + delta only).
// Three kernels: (a) per-block flags + tile sums (one block per thread), (b) one CTA scans
// the tile sums and sets the step record, (c) tile-local scans write the tables.
// ------------------------------------------------------------------------------------
// DIL (fused G2P2G, NEXT N2): the grid of step t+1 built while step t's particles are in
// hand -- a particle of block b moves less than a cell per step, so its step-(t+1) stencil
// lies in blocks b + {-1, 0, 1}^D: touched(b) = some block b + delta, delta in {-1,0,1}^D,
// holds particles at step t.
template <int D, bool DIL = false>
__device__ __forceinline__ void block_flags(const KParams& P, const int* cnt, int gb, int& c,
                                            int& o, int& tch) {
  c = cnt[gb];
  o = c > 0;
  int r = gb / P.nb, bl = gb - r * P.nb;
  int b[D];
  int t = bl;
#pragma unroll
  for (int a = D - 1; a >= 0; --a) { b[a] = t % P.nbpa; t /= P.nbpa; }
  int any = 0;
  if constexpr (DIL) {
#pragma unroll
    for (int dl = 0; dl < Dim<D>::NS; ++dl) {
      int nb_[D], q = dl;
      bool ok = true;
#pragma unroll
      for (int a = D - 1; a >= 0; --a) {
        nb_[a] = b[a] + q % 3 - 1;
        q /= 3;
        ok &= (nb_[a] >= 0) & (nb_[a] < P.nbpa);
      }
      if (ok) any |= __ldg(&cnt[r * P.nb + block_lin<D>(nb_, P.nbpa)]) > 0;
    }
  } else {
#pragma unroll
    for (int dl = 0; dl < (1 << D); ++dl) {
      int nb_[D];
      bool ok = true;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        nb_[a] = b[a] - ((dl >> (D - 1 - a)) & 1);
        ok &= nb_[a] >= 0;
      }
      if (ok) any |= __ldg(&cnt[r * P.nb + block_lin<D>(nb_, P.nbpa)]) > 0;
    }
  }
  tch = any;
}

__device__ __forceinline__ int3 warp_incl_scan3(int3 v) {
  int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int a = __shfl_up_sync(0xffffffffu, v.x, o);
    int b = __shfl_up_sync(0xffffffffu, v.y, o);
    int c = __shfl_up_sync(0xffffffffu, v.z, o);
    if (lane >= o) { v.x += a; v.y += b; v.z += c; }
  }
  return v;
}

__device__ __forceinline__ int4 warp_incl_scan4(int4 v) {
  int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int a = __shfl_up_sync(0xffffffffu, v.x, o);
    int b = __shfl_up_sync(0xffffffffu, v.y, o);
    int c = __shfl_up_sync(0xffffffffu, v.z, o);
    int d = __shfl_up_sync(0xffffffffu, v.w, o);
    if (lane >= o) { v.x += a; v.y += b; v.z += c; v.w += d; }
  }
  return v;
}

// CTA-wide exclusive scan of an int4 (NTH threads)
template <int NTH = kThreads>
__device__ __forceinline__ int4 cta_excl_scan4(int4 v, int4* s_warp, int4& total) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int4 inc = warp_incl_scan4(v);
  if (lane == 31) s_warp[w] = inc;
  __syncthreads();
  if (w == 0) {
    int4 t = lane < NTH / 32 ? s_warp[lane] : make_int4(0, 0, 0, 0);
    int4 ti = warp_incl_scan4(t);
    if (lane < NTH / 32) s_warp[lane] = make_int4(ti.x - t.x, ti.y - t.y, ti.z - t.z, ti.w - t.w);
    if (lane == NTH / 32 - 1) s_warp[NTH / 32] = ti;
  }
  __syncthreads();
  int4 wo = s_warp[w];
  total = s_warp[NTH / 32];
  return make_int4(wo.x + inc.x - v.x, wo.y + inc.y - v.y, wo.z + inc.z - v.z, wo.w + inc.w - v.w);
}

// CTA-wide exclusive scan of an int3 (NTH threads)
template <int NTH = kThreads>
__device__ __forceinline__ int3 cta_excl_scan3(int3 v, int3* s_warp, int3& total) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int3 inc = warp_incl_scan3(v);
  if (lane == 31) s_warp[w] = inc;
  __syncthreads();
  if (w == 0) {
    int3 t = lane < NTH / 32 ? s_warp[lane] : make_int3(0, 0, 0);
    int3 ti = warp_incl_scan3(t);
    if (lane < NTH / 32) s_warp[lane] = make_int3(ti.x - t.x, ti.y - t.y, ti.z - t.z);
    if (lane == NTH / 32 - 1) s_warp[NTH / 32] = ti;
  }
  __syncthreads();
  int3 wo = s_warp[w];
  total = s_warp[NTH / 32];
  return make_int3(wo.x + inc.x - v.x, wo.y + inc.y - v.y, wo.z + inc.z - v.z);
}

// per-tile totals of (count, occupied, touched) -- used once by set_state to size the grid-slot
// arena; flag word of a block: count | occupied << 30 | touched << 31
template <int D, bool DIL = false>
__global__ __launch_bounds__(kScanTile) void k_scan_a(KParams P, const int* __restrict__ cnt,
                                                     unsigned* __restrict__ bflag,
                                                     int3* __restrict__ tile_sums) {
  MPM_PDL_ENTRY();
  __shared__ int3 s_warp[kScanTile / 32 + 1];
  const int gb = blockIdx.x * kScanTile + threadIdx.x;
  int c = 0, o = 0, t = 0;
  if (gb < P.NBT) {
    block_flags<D, DIL>(P, cnt, gb, c, o, t);
    bflag[gb] = (unsigned)c | ((unsigned)o << 30) | ((unsigned)t << 31);
  }
  int3 tot;
  cta_excl_scan3<kScanTile>(make_int3(c, o, t), s_warp, tot);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

// Single-pass binning tables of the step path: one CTA per tile of
// kScanTile blocks, taken in ticket order; block flags -> CTA scan -> decoupled look-back over
// the preceding tiles (aggregate / inclusive prefix published with an epoch-tagged flag, so
// the flags need no reset) -> block_start, occupied list, slot map, touched list.  The grid
// slot of a touched block is checked against the per-step and arena capacities per block; the
// last tile writes the step record (counts, arena base, zeroed work counters).
struct ScanTileState {
  unsigned* flag;          // [n_tiles]: epoch << 2 | status (1 = aggregate, 2 = inclusive prefix)
  int4* agg;               // [n_tiles] (count, big occupied, touched, small occupied)
  int4* incl;              // [n_tiles]
  unsigned long long* ticket;
};

// Outputs in two groups: the binning of step t (block_start, occupied list, info_bin's counts
// and work counters; skipped when info_bin is null) and the grid-slot table of one grid
// (slot map, touched list, info_grid's touched count / arena base; skipped when info_grid is
// null) -- step t's own grid, or with DIL step t+1's (fused G2P2G).  The arena base follows
// the previous grid's slots (info_gprev; null = the segment's first grid, base 0).
template <int D, bool DIL = false>
__global__ __launch_bounds__(kScanTile) void k_scan_lookback(KParams P, const int* __restrict__ cnt, ScanTileState ts,
                                                           unsigned epoch, int n_tiles, int* __restrict__ info_bin,
                                                           int* __restrict__ block_start, int4* __restrict__ occ_list,
                                                           int* __restrict__ info_grid, const int* __restrict__ info_gprev,
                                                           int* __restrict__ slot_of, int* __restrict__ touched_list,
                                                           ErrLatch* err, int t) {
  MPM_PDL_ENTRY();
  __shared__ int4 s_warp[kScanTile / 32 + 1];
  __shared__ int s_tile;
  __shared__ int4 s_pre;
  if (threadIdx.x == 0) s_tile = (int)(atomicAdd(ts.ticket, 1ull) % (unsigned long long)n_tiles);
  __syncthreads();
  const int tile = s_tile;
  const int gb = tile * kScanTile + threadIdx.x;
  int c = 0, o = 0, tc = 0;
  if (gb < P.NBT) block_flags<D, DIL>(P, cnt, gb, c, o, tc);
  // occupied blocks in two classes for the work lists of the block kernels: big ones (at least
  // kBigBlock particles) from the front of occ_list, small ones from its back, so that the CTAs
  // that claim items dynamically take the long items first and the short ones last (a shorter
  // tail when the last items run out)
  const int ob = o && c >= kBigBlock, os = o && c < kBigBlock;
  int4 tot;
  const int4 ex = cta_excl_scan4<kScanTile>(make_int4(c, ob, tc, os), s_warp, tot);
  const unsigned ep = epoch << 2;
  if (threadIdx.x < 32) {  // warp 0: publish, then look back 32 tiles at a time
    const int lane = threadIdx.x;
    if (lane == 0) {
      if (tile == 0) ts.incl[0] = tot; else ts.agg[tile] = tot;
      __threadfence();
      atomicExch(&ts.flag[tile], ep | (tile == 0 ? 2u : 1u));
    }
    int4 pre = make_int4(0, 0, 0, 0);
    for (int i = tile - 1; i >= 0; i -= 32) {
      const int idx = i - lane;
      unsigned f = ep | 2u;  // before tile 0: an empty inclusive prefix
      int4 v = make_int4(0, 0, 0, 0);
      if (idx >= 0) {
        do { f = *((volatile unsigned*)&ts.flag[idx]); } while ((f & ~3u) != ep || (f & 3u) == 0u);
        __threadfence();
        const volatile int* q = (const volatile int*)((f & 3u) == 2u ? &ts.incl[idx] : &ts.agg[idx]);
        v = make_int4(q[0], q[1], q[2], q[3]);
      }
      const unsigned pm = __ballot_sync(0xffffffffu, (f & 3u) == 2u);
      const int stop = pm ? __ffs(pm) - 1 : 31;  // nearest inclusive prefix (lowest lane)
      if (lane > stop) v = make_int4(0, 0, 0, 0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
        v.z += __shfl_xor_sync(0xffffffffu, v.z, o);
        v.w += __shfl_xor_sync(0xffffffffu, v.w, o);
      }
      pre.x += v.x; pre.y += v.y; pre.z += v.z; pre.w += v.w;
      if (pm) break;
    }
    if (lane == 0) {
      if (tile > 0) {
        ts.incl[tile] = make_int4(pre.x + tot.x, pre.y + tot.y, pre.z + tot.z, pre.w + tot.w);
        __threadfence();
        atomicExch(&ts.flag[tile], ep | 2u);
      }
      s_pre = pre;
    }
  }
  __syncthreads();
  const int4 pre = s_pre;
  const int base = info_gprev ? info_gprev[I_BASE] + info_gprev[I_NTOUCH] : 0;
  const int cap = min(P.slots_per_step, P.arena_slots - base);
  if (gb < P.NBT) {
    if (info_bin) {
      block_start[gb] = ex.x + pre.x;
      if (ob) occ_list[ex.y + pre.y] = make_int4(gb, ex.x + pre.x, c, 0);
      if (os) occ_list[P.NBT - 1 - (ex.w + pre.w)] = make_int4(gb, ex.x + pre.x, c, 0);
    }
    if (info_grid) {
      const int sl = ex.z + pre.z;
      const bool fits = tc && sl < cap;
      slot_of[gb] = fits ? base + sl : -1;
      if (fits) touched_list[sl] = gb;
    }
  }
  if (info_bin && gb == P.NBT - 1) block_start[P.NBT] = ex.x + pre.x + c;  // the binned (live) particles
  if (tile == n_tiles - 1 && threadIdx.x == 0) {
    const int ntouch = pre.z + tot.z;
    const int ok = ntouch <= cap;
    if (info_grid) {
      // arena overflow: latched (the forward grows the arena and re-runs from this step); the
      // step still runs on the blocks that got a slot so that every later launch of this call
      // sees consistent tables (its results are discarded)
      if (!ok) latch(err, E_TAPE_FULL, DIL ? t + 1 : t, ntouch);
      info_grid[I_NTOUCH] = ok ? ntouch : max(cap, 0);
      info_grid[I_BASE] = base;
      info_grid[I_OK] = ok;
    }
    if (info_bin) {
      info_bin[I_NOCC] = pre.y + tot.y + pre.w + tot.w;
      info_bin[I_NBIG] = pre.y + tot.y;
      info_bin[I_WORK] = 0;
      info_bin[I_WORK2] = 0;
      info_bin[I_WORK3] = 0;
      info_bin[I_WORK4] = 0;
    }
  }
}

// counting-sort scatter by block (positions inside a block are fixed up by k_block_scatter);
// also zeroes the grid slots of step t (the P2G flush accumulates into them)
__global__ void k_scatter(int NT, const int* __restrict__ key, const int* __restrict__ block_start,
                          int* __restrict__ cnt, int2* __restrict__ tmp_pk, const int* __restrict__ zero_a,
                          const int* __restrict__ zero_b, float4* __restrict__ arena, const int* __restrict__ nslot) {
  MPM_PDL_ENTRY();
  if (nslot) NT = *nslot;  // migrating slab mode: the storage slots of this step (holes have kDeadKey)
  // the grid slots the next scatter accumulates into (zero_a, zero_b: step records or null)
  for (const int* zi : {zero_a, zero_b}) {
    if (!zi) continue;
    const int nz = zi[I_NTOUCH] * kCPB;
    float4* z = arena + (size_t)zi[I_BASE] * kCPB;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nz; i += gridDim.x * blockDim.x)
      z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // kScatQ particles per thread, their key -> block_start loads issued together (the chain
  // key -> block_start -> cursor -> store is latency bound; ILP across particles hides it)
  const int stride = gridDim.x * blockDim.x;
  for (int j0 = blockIdx.x * blockDim.x; j0 < NT; j0 += stride * kScatQ) {  // warp-uniform
    int kj[kScatQ], bs[kScatQ];
#pragma unroll
    for (int q = 0; q < kScatQ; ++q) {
      const int j = j0 + threadIdx.x + q * stride;
      kj[q] = j < NT ? __ldg(&key[j]) : -1;
    }
#pragma unroll
    for (int q = 0; q < kScatQ; ++q) bs[q] = kj[q] >= 0 ? __ldg(&block_start[kj[q] / kCPB]) : 0;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < kScatQ; ++q) {
      const bool valid = kj[q] >= 0;
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      if (valid) {
        const int gb = kj[q] / kCPB;
        const unsigned peers = __match_any_sync(vm, gb);
        const int leader = __ffs(peers) - 1;
        const int n = __popc(peers);
        int old = 0;
        if (lane == leader) old = atomicSub(&cnt[gb], n);
        old = __shfl_sync(peers, old, leader);
        const int rank = __popc(peers & ((1u << lane) - 1));
        tmp_pk[bs[q] + old - n + rank] = make_int2(j0 + threadIdx.x + q * stride, kj[q]);  // (storage index, key)
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// adjoint grid of backward step t: zero its slots and reset the step's work counters.
// Used for the first backward step; later steps are prepared by k_grid_adj of step t+1.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void adj_prepare(int* __restrict__ info_t, float4* __restrict__ g, int tid,
                                            int nthreads) {
  const int n = info_t[I_NTOUCH] * kCPB;
  if (tid == 0) info_t[I_WORK2] = info_t[I_WORK4] = 0;
  for (int i = tid; i < n; i += nthreads) g[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void k_zero_slots(int* __restrict__ info_t, float4* __restrict__ g) {
  MPM_PDL_ENTRY();
  adj_prepare(info_t, g, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// ------------------------------------------------------------------------------------
// Block-tile scatter: P2G (Eqs. 3-5, forward) and G2P^T (step C, adjoint).
//
// One CTA per occupied block (dynamic work counter).  Particles of the block, sorted by
// cell, are turned into a payload by all threads (producer), then thread (cell c, ox)
// accumulates the contributions of its cell's particles to the 3^(D-1) nodes with x
// offset ox in registers (consumer), and writes them into tile copy ox in conflict-free
// phases (no shared-memory atomics).  The 3 copies are summed and each non-zero tile node
// is flushed with one vector RED (red.global.add.v4.f32) into its grid slot.
//
// forward payload:  node value w_o * (A + B o), A = m v - dx G fx, B = dx G, G = -k tau + m C
//                   (Eq. 4 with P_total F^T = tau, k = 4 dt V / dx^2), plus mass w_o m;
// adjoint payload:  A = g_v - B fx, B = 4 res g_C with g_v = dL/dv^{t+1} + dt dL/dx^{t+1}
//                   (step A), g_C = dL/dC^{t+1} + dt dL/dF^{t+1} F^T (step B).
// ------------------------------------------------------------------------------------
template <int D, bool ADJ> struct Pay;
template <int D> struct Pay<D, false> { static constexpr int W = 0, M = 3 * D, A = M + 1, B = A + D, N = B + D * D; };
template <int D> struct Pay<D, true> { static constexpr int W = 0, M = -1, A = 3 * D, B = A + D, N = B + D * D; };
// compact forward payload of the fused G2P2G: the fractional position fx (D rows) in place of
// the 3D stencil weights, which the consumer recomputes (bspl) -- 16 rows instead of 22 in 3D
template <int D> struct PayF { static constexpr int W = 0, M = D, A = D + 1, B = A + D, N = B + D * D; };
template <int D> struct PayFA { static constexpr int W = 0, M = -1, A = D, B = A + D, N = B + D * D; };  // adjoint
template <int D, bool ADJ, bool FX> struct PayOf { using T = Pay<D, ADJ>; };
template <int D> struct PayOf<D, false, true> { using T = PayF<D>; };
template <int D> struct PayOf<D, true, true> { using T = PayFA<D>; };
// quadratic B-spline weight of node offset o at fractional position f (make_stencil's arithmetic)
__device__ __forceinline__ float bspl(float f, int o) {
  const float u = o == 0 ? 1.5f - f : (o == 1 ? f - 1.0f : f - 0.5f);
  return o == 1 ? 0.75f - u * u : 0.5f * u * u;
}

struct StepArgs {
  // forward and adjoint
  const float* st;        // state t (SoA)
  int* perm;              // sorted slot -> storage index (written by forward k_p2g)
  const int2* tmp_pk;     // block-grouped, unsorted (storage index, key) (forward)
  const int* key;         // storage-order keys of step t (forward)
  int* scratch;           // sort scratch for oversize blocks
  const int* orig;        // storage index -> user index, step t
  const float4* prm;      // {m, V, mu, lam} user order
  const int* aid;         // actuator id, user order
  const float* act;       // [B][T][K][D]
  const int* block_start;
  const int4* occ_list;   // occupied-block items {block, first, count, 0} (k_scan_lookback)
  const int* slot_of;
  const int* slot_next;   // fused G2P2G: slot map of grid t+1
  const int* touched_list;
  int* info_t;            // info of step t
  float4* grid;           // tape arena (forward) ; adjoint grid (ADJ)
  const float4* tgrid;    // tape arena (adjoint kernels read the forward grid)
  const float* gin;       // incoming adjoint, storage order t+1 (ADJ)
  float* gout;            // outgoing adjoint, storage order t (ADJ)
  float* st_next;         // state t+1
  int* orig_next;
  int* key_next;          // keys of t+1 (in the single key buffer)
  int* cnt;               // histogram of t+1
  int* info_prev;         // backward: step record of t-1 (its adjoint buffer is prepared)
  float4* agrid_prev;
  float* dmu;             // [NT] user order
  float* dlam;
  float* dmass;           // [NT] user order (NEXT N3)
  float* da;              // [B][T][K][D]
  ErrLatch* err;
  int t;
};


// L2 prefetch of one particle's SoA record (ncomp components at index j) -- issued for a
// block's particles before its tile is staged, so the particle loop's loads hit L2
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
template <int D>
__device__ __forceinline__ void prefetch_record(const float* base, size_t NT, int j, int c0, int ncomp) {
  for (int c = c0; c < c0 + ncomp; ++c) prefetch_l2(base + rix<D>(c, j, NT));
}

// G2P^T's payload carries fx instead of the stencil weights (MPM_SCATA_FX; 15 rows in 3D)
__host__ __device__ constexpr bool scat_fx(bool adj) { return adj ? MPM_SCATA_FX : MPM_SCAT_FX; }
template <int D, bool ADJ>
constexpr int scatter_dyn_smem() {  // payload buffer (forward FX: also the in-block sort, kSortCap ints)
  return (PayOf<D, ADJ, scat_fx(ADJ)>::T::N * kCap > kSortCap || ADJ ? PayOf<D, ADJ, scat_fx(ADJ)>::T::N * kCap : kSortCap) *
         (int)sizeof(float);
}
// payload slot of chunk position p: a warp of consumer threads reads cells whose particles
// sit ~2^d (2D: consecutive cells) or 2^d * {1, 4, 16} (3D thread order below) positions
// apart, which would share 4 banks; the XOR of the low 3 bits with (p >> 5) ^ (p >> 7)
// spreads them over 32.  It permutes every aligned group of 8, so [0, kCap) maps onto itself.
__device__ __forceinline__ int pay_slot(int p) { return p ^ (((p >> 5) ^ (p >> 7)) & 7); }

// Work items of the gathers: (occupied block, part of its particles).  Small problems (fewer
// occupied blocks than CTAs) split each block into up to 8 particle ranges so that more CTAs
// work (each stages its block's tile); large ones keep one item per block.
// i-th occupied block in claim order: the big ones, then the small ones (k_scan_lookback)
// (a record {block, first particle, count, 0}: a claimed item costs one dependent load)
__device__ __forceinline__ int4 occ_item(const KParams& P, const StepArgs& A, int i) {
  const int nbig = A.info_t[I_NBIG];
  return i < nbig ? A.occ_list[i] : A.occ_list[P.NBT - 1 - (i - nbig)];
}

template <bool SPLIT>
__device__ __forceinline__ int work_parts(int n_occ) {
  return SPLIT ? max(1, min(8, (int)gridDim.x / max(n_occ, 1))) : 1;
}
template <bool SPLIT>
__device__ __forceinline__ bool work_item(const KParams& P, const StepArgs& A, int wi, int n_occ, int parts, int& gb, int& s, int& n) {
  if (!SPLIT) {
    if (wi >= n_occ) return false;
    const int4 it = occ_item(P, A, wi);
    gb = it.x;
    s = it.y;
    n = it.z;
    return true;
  }
  if (wi >= n_occ * parts) return false;
  const int bi = wi / parts, part = wi - bi * parts;
  const int4 it = occ_item(P, A, bi);
  gb = it.x;
  const int s0 = it.y, n0 = it.z;
  const int lo = n0 * part / parts, hi = n0 * (part + 1) / parts;
  s = s0 + lo;
  n = hi - lo;
  return true;
}

template <int D>
__device__ __forceinline__ void block_coords(const KParams& P, int gb, int& r, int* bc) {
  r = gb / P.nb;
  int t = gb - r * P.nb;
#pragma unroll
  for (int a = D - 1; a >= 0; --a) { bc[a] = t % P.nbpa; t /= P.nbpa; }
}

// A CTA's next work item, claimed and decoded by thread 0 alone (the block id, particle range,
// rollout and block coordinates, with their runtime divisions) and broadcast through shared
// memory at the claim barrier: the per-item set-up is not repeated by every thread (a block's
// ~512 particles give each thread only ~2 of them, so per-item work is a visible share).
template <int D> struct WorkSh { int gb, s, n, r, bc[D], s0, n0; };  // n < 0: no work left; s0, n0: the whole block
template <int D, bool SPLIT>
__device__ __forceinline__ void claim_item(const KParams& P, const StepArgs& A, int field, int n_occ, int parts,
                                           WorkSh<D>& w) {
  const int wi = atomicAdd(&A.info_t[field], 1);
  int gb, s, n;
  if (!work_item<SPLIT>(P, A, wi, n_occ, parts, gb, s, n)) {
    w.n = -1;
    return;
  }
  w.gb = gb;
  w.s = s;
  w.n = n;
  if (SPLIT) {  // the whole block (its item record again: an L1/L2 hit)
    const int4 it = occ_item(P, A, wi / parts);
    w.s0 = it.y;
    w.n0 = it.z;
  } else {
    w.s0 = s;
    w.n0 = n;
  }
  block_coords<D>(P, gb, w.r, w.bc);
}

// P2G payload of one particle (Eq. 4 with P_total F^T = tau, R1/R21 + actuation S1):
//   B = dx G = -4 res dt V tau + m dx C,  A = m v - B fx   (node value w_o (A + B o))
// t = the step whose actuation applies; latches an inverted element (det F <= 0).
template <int D, int MAT>
__device__ __forceinline__ void p2g_payload(const KParams& P, const StepArgs& A, int r, int t, int u, const float4& pr,
                                            int ai, const float (&v)[D], const float (&H)[D][D],
                                            const float (&Cm)[D][D], const float (&f)[D], float (&Av)[D],
                                            float (&Bm)[D][D]) {
  float sig[D];
#pragma unroll
  for (int a = 0; a < D; ++a)
    sig[a] = ai >= 0 ? P.act_s * A.act[(((size_t)r * P.T + t) * P.K + ai) * D + a] : 0.f;
  const float jm1 = det1m<D>(H);  // J - 1
  if (!(jm1 > -1.f)) latch(A.err, E_INVERTED, t, u);
  const float lnJ = log1pf(jm1);
  float tau[D][D];
  if constexpr (MAT == 1) kirchhoff_fcr<D>(H, pr.z, pr.w, sig, tau, jm1);  // R21
  else kirchhoff_h<D>(H, pr.z, pr.w, sig, tau, lnJ);
  const float kk = 4.f * P.fres * P.dt * pr.y;
  const float mdx = pr.x * P.dx;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) Bm[a][b] = fmaf(-kk, tau[a][b], mdx * Cm[a][b]);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    float acc = pr.x * v[a];
#pragma unroll
    for (int b = 0; b < D; ++b) acc = fmaf(-Bm[a][b], f[b], acc);
    Av[a] = acc;
  }
}

// exclusive scan of the kCPB = 64 cell counts by warp 0: s_cstart[0..64], s_cursor = starts
__device__ __forceinline__ void cell_scan(const int* s_hist, int* s_cstart, int* s_cursor, int tid) {
  static_assert(kCPB == 64, "two cells per lane");
  if (tid < 32) {
    int v0 = s_hist[tid], v1 = s_hist[tid + 32];
    int i0 = v0, i1 = v1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int a = __shfl_up_sync(0xffffffffu, i0, o);
      int b = __shfl_up_sync(0xffffffffu, i1, o);
      if (tid >= o) { i0 += a; i1 += b; }
    }
    int tot0 = __shfl_sync(0xffffffffu, i0, 31);
    s_cstart[tid] = i0 - v0;
    s_cstart[tid + 32] = tot0 + i1 - v1;
    s_cursor[tid] = i0 - v0;
    s_cursor[tid + 32] = tot0 + i1 - v1;
    if (tid == 31) s_cstart[kCPB] = tot0 + i1;
  }
}

// In-place ascending sort of a[0, m) (distinct ints) by the whole CTA: a bitonic network in the
// mirrored form, where every compare-exchange puts the smaller key at the lower index, so the
// virtual +inf padding up to the next power of two never moves and out-of-range partners are
// simply skipped.  O(m log^2 m) work; contains barriers (call uniformly).
__device__ __noinline__ void cta_sort_ints(int* a, int m, int tid, int nthr) {
  int P2 = 1;
  while (P2 < m) P2 <<= 1;
  auto cx = [&](int lo, int hi) {
    if (hi < m) {
      const int x = a[lo], y = a[hi];
      if (y < x) { a[lo] = y; a[hi] = x; }
    }
  };
  for (int k = 2; k <= P2; k <<= 1) {
    for (int i = tid; i < P2 / 2; i += nthr) {  // mirrored merge step of the size-k blocks
      const int h = k / 2, blk = i / h, off = i - blk * h;
      cx(blk * k + off, blk * k + k - 1 - off);
    }
    __syncthreads();
    for (int j = k / 4; j > 0; j >>= 1) {
      for (int i = tid; i < P2 / 2; i += nthr) {
        const int blk = i / j, off = i - blk * j;
        cx(blk * 2 * j + off, blk * 2 * j + off + j);
      }
      __syncthreads();
    }
  }
}

// cells with more particles than this are ordered by cta_sort_ints instead of per-particle
// ranks (O(count) each): a compressed pile-up stays O(n log^2 n) instead of O(n^2)
constexpr int kRankMax = 32;

// the crowded cells of a block: buf (cell-grouped storage indices) sorted per cell into perm
// (out of line: the common path only tests a flag)
__device__ __noinline__ void sort_crowded_cells(int* perm, int* buf, const int* s_cstart, int tid) {
  for (int c = 0; c < kCPB; ++c) {  // uniform: s_cstart is shared
    const int lo = s_cstart[c], hi = s_cstart[c + 1];
    if (hi - lo <= kRankMax) continue;
    cta_sort_ints(buf + lo, hi - lo, tid, kThreads);  // storage indices ascending = stable order
    for (int i = tid; i < hi - lo; i += kThreads) perm[lo + i] = buf[lo + i];
  }
}

// Forward in-block sort (P2G prologue): the block's particles, grouped by k_scatter in
// (storage index, key) pairs, are sorted by (cell, storage index) (stable, R18) into
// perm[s .. s+n); s_cstart gets the cells' ranges.  CTA-wide (contains barriers).
template <int D, bool PF_XF = false>
__device__ __forceinline__ bool block_cell_sort(const KParams& P, const StepArgs& A, int s, int n, int tid,
                                                int* s_hist, int* s_cstart, int* s_cursor, int* s_sort,
                                                int* s_pout = nullptr) {
  const size_t NT = P.NT;
  // (storage index, cell) of this thread's first two particles stay in registers
  int pj[2] = {0, 0}, pc[2] = {0, 0};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int i = tid + q * kThreads;
    if (i < n) {
      const int2 e = A.tmp_pk[s + i];
      pj[q] = e.x;
      pc[q] = e.y & (kCPB - 1);
      atomicAdd(&s_hist[pc[q]], 1);
#if MPM_SCAT_PF
      // the producer reads this particle's record after the sort: start fetching it now
      // (PF_XF: the fused G2P2G reads x and F only)
      if (PF_XF) {
        prefetch_record<D>(A.st, NT, e.x, 0, D);
        prefetch_record<D>(A.st, NT, e.x, comp_F<D>(0, 0), D * D);
      } else {
        prefetch_record<D>(A.st, NT, e.x, 0, Dim<D>::S);
      }
      prefetch_l2(&A.orig[e.x]);
#endif
    }
  }
  for (int i = tid + 2 * kThreads; i < n; i += kThreads) atomicAdd(&s_hist[A.tmp_pk[s + i].y & (kCPB - 1)], 1);
  __syncthreads();
  __shared__ int s_crowd;  // some cell holds more than kRankMax particles (a pile-up)
  cell_scan(s_hist, s_cstart, s_cursor, tid);
  if (tid < 32) {
    const bool cr = __any_sync(0xffffffffu, (s_hist[tid] > kRankMax) | (s_hist[tid + 32] > kRankMax));
    if (tid == 0) s_crowd = cr;
  }
  __syncthreads();
  const bool crowd = s_crowd;
  int* buf = (n <= kSortCap) ? s_sort : (A.scratch + s);
#pragma unroll
  for (int q = 0; q < 2; ++q)
    if (tid + q * kThreads < n) {
      const int at = atomicAdd(&s_cursor[pc[q]], 1);
      MPM_CHECK(at >= 0 && at < n);
      buf[at] = pj[q];
    }
  for (int i = tid + 2 * kThreads; i < n; i += kThreads) {
    const int2 e = A.tmp_pk[s + i];
    buf[atomicAdd(&s_cursor[e.y & (kCPB - 1)], 1)] = e.x;
  }
  __syncthreads();
  // rank of each particle among its cell's (stable: ties by storage index, R18), per input
  // element: the first two of a thread still hold (storage index, cell) in registers, the
  // others re-read their (storage index, key) pair -- no search for the cell of a position
  auto place = [&](int j, int c) {
    const int lo = s_cstart[c], hi = s_cstart[c + 1];
    if (crowd && hi - lo > kRankMax) return;  // a crowded cell: sorted below
    int rank = 0;
#pragma unroll 4
    for (int q = lo; q < hi; ++q) rank += buf[q] < j;
    A.perm[s + lo + rank] = j;
    if (s_pout && lo + rank < kCapPerm) s_pout[lo + rank] = j;  // the caller's shared copy
  };
#pragma unroll
  for (int q = 0; q < 2; ++q)
    if (tid + q * kThreads < n) place(pj[q], pc[q]);
  for (int i = tid + 2 * kThreads; i < n; i += kThreads) {
    const int2 e = A.tmp_pk[s + i];
    place(e.x, e.y & (kCPB - 1));
  }
  if (crowd) sort_crowded_cells(A.perm + s, buf, s_cstart, tid);
  __syncthreads();
  return crowd;  // uniform; crowded cells are not in s_pout
}

// Scatter consumer: thread (ox, c), c = cell, accumulates the NSUB nodes c + (ox, *) of the
// payload positions [i0, i1) (ORD: through the order s_ord) in registers, then writes them
// into tile copy ox in NSUB conflict-free phases (64-thread named barriers).
template <int D, bool ADJ, bool ORD, int CAP = kCap, bool FX = false>
__device__ __forceinline__ void scatter_consume(const float (*s_pay)[CAP], float4 (*s_tile)[Dim<D>::TN], int i0,
                                                int i1, const short* s_ord, int ox, int c, int tid) {
  using PY = typename PayOf<D, ADJ, FX>::T;
  constexpr int BB = Dim<D>::BB, TE = Dim<D>::TE;
  constexpr int NSUB = (D == 3) ? 9 : 3;
  // consumer: thread (ox, c), c = cell, accumulates NSUB nodes
  float4 acc[NSUB];
#pragma unroll
  for (int q = 0; q < NSUB; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (tid < 3 * kCPB) {
    for (int i0s = i0; i0s < i1; ++i0s) {
      const int i = pay_slot(ORD ? (int)s_ord[i0s] : i0s);
      // stencil weights: stored (W rows, 3 per axis) or recomputed from fx (FX: 1 row per axis)
      float wyv[3], wzv[3];
#pragma unroll
      for (int o = 0; o < 3; ++o) {
        wyv[o] = FX ? bspl(s_pay[PY::W + 1][i], o) : s_pay[PY::W + 3 + o][i];
        wzv[o] = D == 3 ? (FX ? bspl(s_pay[PY::W + 2 % D][i], o) : s_pay[PY::W + 6 % (3 * D) + o][i]) : 0.f;
      }
      const float wx = FX ? bspl(s_pay[PY::W][i], ox) : s_pay[PY::W + ox][i];
      float Ax[3];
#pragma unroll
      for (int a = 0; a < D; ++a) Ax[a] = s_pay[PY::A + a][i] + (float)ox * s_pay[PY::B + a * D + 0][i];
      const float mp = ADJ ? 0.f : s_pay[PY::M < 0 ? 0 : PY::M][i];
      if (D == 3) {
        float B1[3], B2[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) { B1[a] = s_pay[PY::B + a * D + 1][i]; B2[a] = s_pay[PY::B + a * D + 2 % D][i]; }
#pragma unroll
        for (int oy = 0; oy < 3; ++oy) {
          const float wxy = wx * wyv[oy];
#if MPM_FFMA2_SCAT
          // node value A + oy B1 + oz B2 and the accumulation as packed fp32x2 FMAs:
          // (x, y) and (z, m) pairs (sm_100 FFMA2; per component the same fused op)
          const float2 rxy = __ffma2_rn(make_float2((float)oy, (float)oy), make_float2(B1[0], B1[1]),
                                        make_float2(Ax[0], Ax[1]));
          const float rz = fmaf((float)oy, B1[2], Ax[2]);
#pragma unroll
          for (int oz = 0; oz < 3; ++oz) {
            const float W = wxy * wzv[oz];
            float4& q = acc[oy * 3 + oz];
            const float2 vxy = oz ? __ffma2_rn(make_float2((float)oz, (float)oz), make_float2(B2[0], B2[1]), rxy) : rxy;
            const float vz = oz ? fmaf((float)oz, B2[2], rz) : rz;
            const float2 qxy = __ffma2_rn(make_float2(W, W), vxy, make_float2(q.x, q.y));
            const float2 qzw = __ffma2_rn(make_float2(W, W), make_float2(vz, ADJ ? 0.f : mp), make_float2(q.z, q.w));
            q = make_float4(qxy.x, qxy.y, qzw.x, ADJ ? q.w : qzw.y);
          }
#else
#pragma unroll
          for (int oz = 0; oz < 3; ++oz) {
            const float W = wxy * wzv[oz];
            float4& q = acc[oy * 3 + oz];
            q.x = fmaf(W, Ax[0] + (float)oy * B1[0] + (float)oz * B2[0], q.x);
            q.y = fmaf(W, Ax[1] + (float)oy * B1[1] + (float)oz * B2[1], q.y);
            q.z = fmaf(W, Ax[2] + (float)oy * B1[2] + (float)oz * B2[2], q.z);
            if (!ADJ) q.w = fmaf(W, mp, q.w);
          }
#endif
        }
      } else {
        float B1[2];
#pragma unroll
        for (int a = 0; a < 2; ++a) B1[a] = s_pay[PY::B + a * D + 1][i];
#pragma unroll
        for (int oy = 0; oy < 3; ++oy) {
          const float W = wx * wyv[oy];
          float4& q = acc[oy];
          q.x = fmaf(W, Ax[0] + (float)oy * B1[0], q.x);
          q.y = fmaf(W, Ax[1] + (float)oy * B1[1], q.y);
          if (!ADJ) q.w = fmaf(W, mp, q.w);
        }
      }
    }
  }
  // phase-write: in phase q the 64 threads of copy ox write the distinct nodes c + (ox, q);
  // only threads of the same copy can collide across phases -> 64-thread named barriers
  if (tid < 3 * kCPB) {
    int cc[D];
    {
      int t = c;
#pragma unroll
      for (int a = D - 1; a >= 0; --a) { cc[a] = t % BB; t /= BB; }
    }
#pragma unroll
    for (int q = 0; q < NSUB; ++q) {
      int tl;
      if (D == 3) tl = ((cc[0] + ox) * TE + cc[1] + q / 3) * TE + cc[D - 1] + q % 3;
      else tl = (cc[0] + ox) * TE + cc[D - 1] + q;
      MPM_CHECK(tl >= 0 && tl < Dim<D>::TN);
      float4 v = s_tile[ox][tl];
      v.x += acc[q].x; v.y += acc[q].y; v.z += acc[q].z; v.w += acc[q].w;
      s_tile[ox][tl] = v;
      if (q + 1 < NSUB) asm volatile("bar.sync %0, %1;" ::"r"(1 + ox), "r"(kCPB) : "memory");
    }
  }
}

// Scatter flush: the 3 tile copies summed, one vector RED (red.global.add.v4.f32) per
// non-zero node into its grid slot; myslot (lanes 0..2^D-1) = the slots of blocks bc + {0,1}^D.
template <int D, bool ADJ>
__device__ __forceinline__ void scatter_flush(const KParams& P, float4* grid, const float4 (*s_tile)[Dim<D>::TN],
                                              const int* bc, int myslot, int base_slot, int tid) {
  constexpr int BB = Dim<D>::BB, TE = Dim<D>::TE, TN = Dim<D>::TN;
  for (int t0 = 0; t0 < TN; t0 += kThreads) {  // uniform trip count: whole warps reach the shuffle
    const int tn = t0 + tid;
    int tl[D], sb = 0;
    {
      int t = tn;
#pragma unroll
      for (int a = D - 1; a >= 0; --a) {
        tl[a] = t % TE;
        sb |= (tl[a] >= BB) << (D - 1 - a);
        t /= TE;
      }
    }
    const int slot = __shfl_sync(0xffffffffu, myslot, sb);
    if (tn >= TN) continue;
    float4 v0 = s_tile[0][tn], v1 = s_tile[1][tn], v2 = s_tile[2][tn];
    float4 v = make_float4(v0.x + v1.x + v2.x, v0.y + v1.y + v2.y, v0.z + v1.z + v2.z, v0.w + v1.w + v2.w);
    if (v.x == 0.f && v.y == 0.f && v.z == 0.f && v.w == 0.f) continue;
    int loc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) loc[a] = (bc[a] * BB + tl[a]) & (BB - 1);
    if (slot < 0) continue;  // outside the domain / untouched (cannot happen for non-zero nodes)
    float4* dst = grid + (size_t)(ADJ ? slot - base_slot : slot) * kCPB + cell_lin<D>(loc);
    atomicAdd(dst, v);  // red.global.add.v4.f32
  }
}

template <int D, bool ADJ, int MAT = 0, bool SPLIT = false>
__global__ __launch_bounds__(kThreads, ADJ ? MPM_SCATA_MINB : MPM_SCAT_MINB) void k_block_scatter(KParams P, StepArgs A) {
  MPM_PDL_ENTRY();
  using DD = Dim<D>;
  constexpr bool FX = scat_fx(ADJ);
  using PY = typename PayOf<D, ADJ, FX>::T;
  constexpr int BB = DD::BB, TN = DD::TN;
  __shared__ int s_hist[kCPB];
  __shared__ int s_cstart[kCPB + 1];
  __shared__ int s_cursor[kCPB];
  __shared__ int s_sort_st[(ADJ || scat_fx(ADJ)) ? 1 : kSortCap];  // forward FX: the sort uses the payload area
  extern __shared__ __align__(16) unsigned char s_dyn[];
  float (*s_pay)[kCap] = reinterpret_cast<float (*)[kCap]>(s_dyn);  // [PY::N][kCap], dynamic
  int* s_sort = scat_fx(ADJ) ? reinterpret_cast<int*>(s_dyn) : s_sort_st;  // done before the payload is written
  __shared__ float4 s_tile[3][TN];
  __shared__ WorkSh<D> s_w;
  const int tid = threadIdx.x;
  const size_t NT = P.NT;
  const int work_field = ADJ ? I_WORK2 : I_WORK;
  const int n_occ = A.info_t[I_NOCC];
  const int base_slot = A.info_t[I_BASE];

  // SPLIT (adjoint only; the forward sorts whole blocks): small problems give a block's
  // particle ranges to several CTAs, each flushing its own partial tile with REDs
  static_assert(!SPLIT || ADJ, "only the adjoint scatter splits blocks");
  const int parts = work_parts<SPLIT>(n_occ);
  for (;;) {
    if (tid == 0) claim_item<D, SPLIT>(P, A, work_field, n_occ, parts, s_w);
    __syncthreads();
    const int n = s_w.n;
    if (n < 0) break;
    if (SPLIT && n == 0) {  // uniform; every thread has read s_w before thread 0 claims again
      __syncthreads();
      continue;
    }
    const int gb = s_w.gb, s = s_w.s, r = s_w.r;
    int bc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) bc[a] = s_w.bc[a];
    // the tile's 2^D block slots (flush): looked up now, used at the end
    int myslot = -1;
    {
      const int lane = tid & 31;
      if (lane < (1 << D)) {
        int nb_[D];
        bool inside = true;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          nb_[a] = bc[a] + ((lane >> (D - 1 - a)) & 1);
          inside &= nb_[a] < P.nbpa;
        }
        if (inside) myslot = __ldg(&A.slot_of[r * P.nb + block_lin<D>(nb_, P.nbpa)]);
      }
    }
    if (tid < kCPB) {
      s_hist[tid] = 0;
      if (ADJ) { s_cstart[tid] = 0x7fffffff; s_cursor[tid] = -1; }  // per-chunk [first, last] of a cell
    }
    for (int i = tid; i < 3 * TN; i += kThreads) (&s_tile[0][0])[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();

    if (!ADJ) block_cell_sort<D>(P, A, s, n, tid, s_hist, s_cstart, s_cursor, s_sort);

    // ---- chunks of kCap particles: produce payload, consume per (cell, ox), phase-write ----
    // consumer thread -> (ox, cell).  3D: cell z fastest, then x, then y, so the 8 threads of a
    // quarter-warp write tile nodes 36 float4 apart in x (conflict-free 128-bit phase writes)
    const int ox = tid / kCPB;
    const int c = D == 3 ? ((((tid >> 2) & 3) * 4 + ((tid >> 4) & 3)) * 4 + (tid & 3)) : tid % kCPB;
    for (int lo = 0; lo < n; lo += kCap) {
      const int hi = min(n, lo + kCap);
      if (ADJ && lo > 0) {  // later chunks of an oversize block: reset the cell sub-ranges
        if (tid < kCPB) { s_cstart[tid] = 0x7fffffff; s_cursor[tid] = -1; }
        __syncthreads();
      }
      for (int pi = tid; pi < hi - lo; pi += kThreads) {
        const int k = s + lo + pi;
        const int j = A.perm[k];
        float x[D], f[D];
        Stencil<D> sc;
#pragma unroll
        for (int a = 0; a < D; ++a) x[a] = A.st[rix<D>(comp_x<D>(a), j, NT)];
        make_stencil<D>(x, P.fres, sc);
        const int ps = pay_slot(pi);
        MPM_CHECK(ps >= 0 && ps < kCap);
#pragma unroll
        for (int a = 0; a < D; ++a) {
          f[a] = sc.fx[a];
          if (FX) {
            s_pay[PY::W + a][ps] = sc.fx[a];
          } else {
#pragma unroll
            for (int o = 0; o < 3; ++o) s_pay[PY::W + a * 3 + o][ps] = sc.w[a][o];
          }
        }
        if (ADJ) {
          int cl[D];
#pragma unroll
          for (int a = 0; a < D; ++a) cl[a] = sc.base[a] & (BB - 1);
          atomicMin(&s_cstart[cell_lin<D>(cl)], pi);
          atomicMax(&s_cursor[cell_lin<D>(cl)], pi);
        }
        float Av[D], Bm[D][D];
        if (!ADJ) {
          const int u = A.orig[j];
          const float4 pr = A.prm[u];  // m, V, mu, lam
          float H[D][D], Cm[D][D], v[D];
#pragma unroll
          for (int a = 0; a < D; ++a) {
            v[a] = A.st[rix<D>(comp_v<D>(a), j, NT)];
#pragma unroll
            for (int b = 0; b < D; ++b) {
              H[a][b] = A.st[rix<D>(comp_F<D>(a, b), j, NT)];
              Cm[a][b] = A.st[rix<D>(comp_C<D>(a, b), j, NT)];
            }
          }
          p2g_payload<D, MAT>(P, A, r, A.t, u, pr, A.aid[u], v, H, Cm, f, Av, Bm);
          if (PY::M >= 0) s_pay[PY::M < 0 ? 0 : PY::M][ps] = pr.x;
        } else {
          // steps A and B: g_v = gv + dt gx ; g_C = gC + dt gF F^T
          const float* gi = A.gin;
          float F[D][D], gF[D][D], gC[D][D], gv[D];
#pragma unroll
          for (int a = 0; a < D; ++a) {
            gv[a] = fmaf(P.dt, gi[rix<D>(comp_x<D>(a), k, NT)], gi[rix<D>(comp_v<D>(a), k, NT)]);
#pragma unroll
            for (int b = 0; b < D; ++b) {
              F[a][b] = A.st[rix<D>(comp_F<D>(a, b), j, NT)] + (a == b ? 1.f : 0.f);  // F = I + H
              gF[a][b] = gi[rix<D>(comp_F<D>(a, b), k, NT)];
              gC[a][b] = gi[rix<D>(comp_C<D>(a, b), k, NT)];
            }
          }
          const float s4 = 4.f * P.fres;
#pragma unroll
          for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = 0; b < D; ++b) {
              float acc = gC[a][b];
#pragma unroll
              for (int c = 0; c < D; ++c) acc = fmaf(P.dt * gF[a][c], F[b][c], acc);
              Bm[a][b] = s4 * acc;
            }
#pragma unroll
          for (int a = 0; a < D; ++a) {
            float acc = gv[a];
#pragma unroll
            for (int b = 0; b < D; ++b) acc = fmaf(-Bm[a][b], f[b], acc);
            Av[a] = acc;
          }
        }
#pragma unroll
        for (int a = 0; a < D; ++a) {
          s_pay[PY::A + a][ps] = Av[a];
#pragma unroll
          for (int b = 0; b < D; ++b) s_pay[PY::B + a * D + b][ps] = Bm[a][b];
        }
      }
      __syncthreads();

      {
        const int i0 = (tid < 3 * kCPB) ? (ADJ ? s_cstart[c] : max(s_cstart[c], lo) - lo) : 0;
        const int i1 = (tid < 3 * kCPB) ? (ADJ ? s_cursor[c] + 1 : min(s_cstart[c + 1], hi) - lo) : 0;
        scatter_consume<D, ADJ, false, kCap, FX>(s_pay, s_tile, i0, i1, nullptr, ox, c, tid);
      }
      __syncthreads();  // payload consumed, tile copies written
    }

    // ---- flush: one vector RED per non-zero tile node.  The tile spans the 2^D blocks
    //      bc + {0, 1}^D: lanes 0..2^D-1 of each warp look their slots up, nodes take theirs by
    //      shuffle (one dependent global load less per node) ----
    scatter_flush<D, ADJ>(P, A.grid, s_tile, bc, myslot, base_slot, tid);
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------
// The grid operation (Eq. 6; gravity R5; wall projection R6) has no kernel of its
// own: the memo keeps the (p, m) P2G accumulated, and every gather computes
// vbar = p / m + dt g and the projection per node while staging its tile (fetch_node).
// ------------------------------------------------------------------------------------


// ------------------------------------------------------------------------------------
// Block-tile gathers (G2P, P2G^T).  One CTA per occupied grid block (dynamic work
// counter).  The block's (Bb+2)^D node tile is staged once in shared memory -- node
// velocity after the wall projection of step L (applied once per node), and
// for P2G^T also the adjoint node (dL/dp_i, dL/dm_i) -- then every particle of the block
// (contiguous in sorted order) reads its 3^D stencil from the tile.
// Weights are separable, W = wx(ox) wy(oy) wz(oz); oz-sums are formed first and folded
// per (ox, oy), so the moments sum_i W v_i o_b cost O(1) per node.
// ------------------------------------------------------------------------------------

template <int D, bool TWO, bool RAW = false>
__device__ __forceinline__ void fetch_node_slot(const KParams& P, const StepArgs& A, const int* node, int slot,
                                                size_t abase, float4& v, float4& ad);

// fetch one node of step t: velocity after the wall projection (v.w = m) and, optionally,
// the adjoint node (dL/dp_i, dL/dm_i); zero outside the domain / untouched blocks
template <int D, bool TWO>
__device__ __forceinline__ void fetch_node(const KParams& P, const StepArgs& A, int r, const int* node,
                                           size_t abase, float4& v, float4& ad) {
  using DD = Dim<D>;
  int nb_[D], loc[D];
  bool inside = true;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    inside &= node[a] < P.res;
    nb_[a] = node[a] >> DD::LOG_BB;
    loc[a] = node[a] & (DD::BB - 1);
  }
  v = make_float4(0.f, 0.f, 0.f, 0.f);
  ad = v;
  if (!inside) return;
  fetch_node_slot<D, TWO>(P, A, node, __ldg(&A.slot_of[r * P.nb + block_lin<D>(nb_, P.nbpa)]), abase, v, ad);
}

// the same with the node's grid slot already known (-1: untouched block)
template <int D, bool TWO, bool RAW>
__device__ __forceinline__ void fetch_node_slot(const KParams& P, const StepArgs& A, const int* node, int slot,
                                                size_t abase, float4& v, float4& ad) {
  using DD = Dim<D>;
  int loc[D];
#pragma unroll
  for (int a = 0; a < D; ++a) loc[a] = node[a] & (DD::BB - 1);
  v = make_float4(0.f, 0.f, 0.f, 0.f);
  ad = v;
  if (slot < 0) return;
  const size_t addr = (size_t)slot * kCPB + cell_lin<D>(loc);
  MPM_CHECK(slot < P.arena_slots);
  const float4 pm = A.tgrid[addr];  // (p, m) as accumulated by P2G -- the memo's grid
  if (!(pm.w > 0.f)) return;        // empty node: v = 0 (R13), no adjoint
  // grid operation (Eq. 6 + gravity, R5): vbar = p / m + dt g, then the wall projection (R6)
  float vb[D], vv[D];
  vb[0] = pm.x / pm.w + P.dt * P.g[0];
  vb[1] = pm.y / pm.w + P.dt * P.g[1];
  if constexpr (D == 3) vb[2] = pm.z / pm.w + P.dt * P.g[2];
#pragma unroll
  for (int a = 0; a < D; ++a) vv[a] = vb[a];
  if (in_band<D>(node, P.res, P.bound)) project_node<D>(vv, node, P);
  v = make_float4(vv[0], vv[1], D == 3 ? vv[D - 1] : 0.f, pm.w);
  if (TWO) {
    ad = A.grid[addr - abase];
    if constexpr (RAW) {
    // gridT (steps L, D, E; what k_grid_adj computes in place) on the raw dL/dvbar that G2P^T
    // accumulated: the wall projection's adjoint, then vbar = p/m + dt g -> dL/dp = gv / m,
    // dL/dm = -(p/m . gv) / m
    const float im = 1.f / pm.w;
    float vg[D], gv[D];
    vg[0] = fmaf(pm.x, im, P.dt * P.g[0]); vg[1] = fmaf(pm.y, im, P.dt * P.g[1]);
    gv[0] = ad.x; gv[1] = ad.y;
    if constexpr (D == 3) { vg[2] = fmaf(pm.z, im, P.dt * P.g[2]); gv[2] = ad.z; }
    if (in_band<D>(node, P.res, P.bound)) project_node_adj<D>(vg, gv, node, P);
    float pg = 0.f;
#pragma unroll
    for (int d = 0; d < D; ++d) pg = fmaf(vg[d] - P.dt * P.g[d], gv[d], pg);
    ad = make_float4(gv[0] * im, gv[1] * im, D == 3 ? gv[D - 1] * im : 0.f, -pg * im);
    }
  }
}

// Stage the block's node tile: s_v = v_i - vref, s_a = a_i - aref, with (vref, aref) the
// values of the block-centre node.  Every stencil sum the gathers form is invariant under
// such a constant shift (sum W = 1, sum W o = fx, sum dW = 0, sum dW (o - fx)^T = res I for
// the quadratic B-spline); the shift removes the common-mode velocity / adjoint so the fp32
// cancellations in C' (Eq. 8) and in step J shrink to |v_i - vref|.  Callers add the
// references back where an unshifted sum is needed (v' = S + vref, sum W dp = S_d + aref).
template <int D, bool TWO, int NTH = kThreads, bool RAW = false>
__device__ __forceinline__ void stage_tile(const KParams& P, const StepArgs& A, int r, const int* bc,
                                           float4* s_v, float4* s_a, size_t abase, float4& vref,
                                           float4& aref) {
  using DD = Dim<D>;
  // the tile's nodes lie in the 2^D blocks bc + {0, 1}^D (TE = BB + 2 <= 2 BB): lanes 0..2^D-1
  // of every warp look their grid slots up once and each node takes its slot by shuffle, so a
  // node costs one global load instead of a dependent pair (no barrier needed)
  const int lane = threadIdx.x & 31;
  int myslot = -1;
  if (lane < (1 << D)) {
    int nb_[D];
    bool inside = true;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      nb_[a] = bc[a] + ((lane >> (D - 1 - a)) & 1);
      inside &= nb_[a] < P.nbpa;
    }
    if (inside) myslot = __ldg(&A.slot_of[r * P.nb + block_lin<D>(nb_, P.nbpa)]);
  }
  {
    int node[D];
#pragma unroll
    for (int a = 0; a < D; ++a) node[a] = bc[a] * DD::BB + DD::BB / 2;
    fetch_node_slot<D, TWO, RAW>(P, A, node, __shfl_sync(0xffffffffu, myslot, 0), abase, vref, aref);
  }
  for (int t0 = 0; t0 < DD::TN; t0 += NTH) {  // uniform trip count: whole warps reach the shuffle
    const int tn = t0 + (int)threadIdx.x;
    int node[D], sb = 0;
    int t = tn;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      const int l = t % DD::TE;
      node[a] = bc[a] * DD::BB + l;
      sb |= (l >= DD::BB) << (D - 1 - a);
      t /= DD::TE;
    }
    const int slot = __shfl_sync(0xffffffffu, myslot, sb);
    if (tn < DD::TN) {
      float4 v, ad;
      fetch_node_slot<D, TWO, RAW>(P, A, node, slot, abase, v, ad);
      s_v[tn] = make_float4(v.x - vref.x, v.y - vref.y, v.z - vref.z, v.w);
      if (TWO) s_a[tn] = make_float4(ad.x - aref.x, ad.y - aref.y, ad.z - aref.z, ad.w - aref.w);
    }
  }
}

template <int D, int OX, int OY, int OZ>
__device__ __forceinline__ int tile_idx(const int* lb) {
  constexpr int TE = Dim<D>::TE;
#pragma unroll
  for (int a = 0; a < D; ++a) MPM_CHECK(lb[a] >= 0 && lb[a] <= TE - 3);  // stencil inside the tile
  if constexpr (D == 3) return ((lb[0] + OX) * TE + lb[1] + OY) * TE + lb[2] + OZ;
  else return (lb[0] + OX) * TE + lb[1] + OY;
}

// ---- G2P (Eqs. 7-10): v' = S, C' = 4 res (M - S fx^T), F' = (I + dt C') F,
//      x' = x + dt v'; writes state t+1 in sorted order + keys/histogram of step t+1 ----
template <int D, int OX, int OY, int OZ>
__device__ __forceinline__ void g2p_node(const float4* s_v, const int* lb, const Stencil<D>& sc,
                                         const float4& vref, float wxy, float* Sxy, float* Zxy) {
  const float4 g = s_v[tile_idx<D, OX, OY, OZ>(lb)];
  float vi[3] = {g.x, g.y, g.z};
  const float W = (D == 3) ? wxy * sc.w[D - 1][OZ] : wxy;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const float wv = W * vi[a];
    Sxy[a] += wv;
    if (OZ == 1) Zxy[a] += wv;
    if (OZ == 2) Zxy[a] = fmaf(2.f, wv, Zxy[a]);
  }
}

template <int D, int OX, int OY>
__device__ __forceinline__ void g2p_row(const float4* s_v, const int* lb, const Stencil<D>& sc,
                                        const float4& vref, float* S, float (&M)[D][D]) {
  const float wxy = sc.w[0][OX] * sc.w[1][OY];
  if constexpr (D == 3 && MPM_FFMA2) {
    // row sums a0 = sum_oz wz v, a1 = sum_oz oz wz v with packed fp32x2 FMAs on (x, y)
    // (sm_100 FFMA2: per component the same fused op as fmaf), z as scalar FMAs
    float2 a0 = make_float2(0.f, 0.f), a1 = a0;
    float a0z = 0.f, a1z = 0.f;
#pragma unroll
    for (int oz = 0; oz < 3; ++oz) {
      const float4 g = s_v[tile_idx<D, OX, OY, 0>(lb) + oz];
      const float wz = sc.w[2][oz];
      const float2 vxy = make_float2(g.x, g.y);
      a0 = __ffma2_rn(make_float2(wz, wz), vxy, a0);
      a0z = fmaf(wz, g.z, a0z);
      if (oz) {
        const float ow = (float)oz * wz;
        a1 = __ffma2_rn(make_float2(ow, ow), vxy, a1);
        a1z = fmaf(ow, g.z, a1z);
      }
    }
    const float2 w2 = make_float2(wxy, wxy);
    float2 sxy = __ffma2_rn(w2, a0, make_float2(S[0], S[1]));
    S[0] = sxy.x; S[1] = sxy.y; S[2] = fmaf(wxy, a0z, S[2]);
    if (OX) {
      const float2 m = __ffma2_rn(make_float2((float)OX * wxy, (float)OX * wxy), a0, make_float2(M[0][0], M[1][0]));
      M[0][0] = m.x; M[1][0] = m.y; M[2][0] = fmaf((float)OX * wxy, a0z, M[2][0]);
    }
    if (OY) {
      const float2 m = __ffma2_rn(make_float2((float)OY * wxy, (float)OY * wxy), a0, make_float2(M[0][1], M[1][1]));
      M[0][1] = m.x; M[1][1] = m.y; M[2][1] = fmaf((float)OY * wxy, a0z, M[2][1]);
    }
    {
      const float2 m = __ffma2_rn(w2, a1, make_float2(M[0][2], M[1][2]));
      M[0][2] = m.x; M[1][2] = m.y; M[2][2] = fmaf(wxy, a1z, M[2][2]);
    }
  } else {
    float Sxy[D], Zxy[D];
#pragma unroll
    for (int a = 0; a < D; ++a) Sxy[a] = Zxy[a] = 0.f;
    if constexpr (D == 3) {
      g2p_node<D, OX, OY, 0>(s_v, lb, sc, vref, wxy, Sxy, Zxy);
      g2p_node<D, OX, OY, 1>(s_v, lb, sc, vref, wxy, Sxy, Zxy);
      g2p_node<D, OX, OY, 2>(s_v, lb, sc, vref, wxy, Sxy, Zxy);
    } else {
      g2p_node<D, OX, OY, 0>(s_v, lb, sc, vref, wxy, Sxy, Zxy);
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {
      S[a] += Sxy[a];
      if (OX) M[a][0] = fmaf((float)OX, Sxy[a], M[a][0]);
      if (OY) M[a][1] = fmaf((float)OY, Sxy[a], M[a][1]);
      if constexpr (D == 3) M[a][2] += Zxy[a];
    }
  }
}

// G2P of the particle at sorted position k (Eqs. 7-10): writes state t+1 at k, its user
// index, key and the block histogram of step t+1; returns the new x, v, C and H = F - I in
// registers (the fused G2P2G scatters them) and whether the new base index is valid.
// COH: perm was written by this kernel (the fused sort) -- a coherent load, not the
// read-only path.
template <int D, bool COH = false, bool PRM = false>
__device__ __forceinline__ bool g2p_particle(const KParams& P, const StepArgs& A, const float4* s_v,
                                             const float4& vref, const int* bc, int r, int k, float (&x)[D],
                                             float (&vn)[D], float (&Cn)[D][D], float (&Hn)[D][D], int& u,
                                             float4* pr = nullptr, int* ai = nullptr, int j_in = -1) {
  const size_t NT = P.NT;
  const int j = j_in >= 0 ? j_in : COH ? __ldcg(&A.perm[k]) : __ldg(&A.perm[k]);
  float H[D][D];  // H = F - I
#pragma unroll
  for (int a = 0; a < D; ++a) {
    x[a] = __ldg(&A.st[rix<D>(comp_x<D>(a), j, NT)]);
#pragma unroll
    for (int b = 0; b < D; ++b) H[a][b] = __ldg(&A.st[rix<D>(comp_F<D>(a, b), j, NT)]);
  }
  u = __ldg(&A.orig[j]);
  if (PRM) {  // the fused P2G's parameters: issued now, consumed after the gather
    *pr = __ldg(&A.prm[u]);
    *ai = __ldg(&A.aid[u]);
  }
  Stencil<D> sc;
  make_stencil<D>(x, P.fres, sc);
  int lb[D];
#pragma unroll
  for (int a = 0; a < D; ++a) lb[a] = sc.base[a] - bc[a] * Dim<D>::BB;
  float S[D], M[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    S[a] = 0.f;
#pragma unroll
    for (int b = 0; b < D; ++b) M[a][b] = 0.f;
  }
  g2p_row<D, 0, 0>(s_v, lb, sc, vref, S, M); g2p_row<D, 0, 1>(s_v, lb, sc, vref, S, M); g2p_row<D, 0, 2>(s_v, lb, sc, vref, S, M);
  g2p_row<D, 1, 0>(s_v, lb, sc, vref, S, M); g2p_row<D, 1, 1>(s_v, lb, sc, vref, S, M); g2p_row<D, 1, 2>(s_v, lb, sc, vref, S, M);
  g2p_row<D, 2, 0>(s_v, lb, sc, vref, S, M); g2p_row<D, 2, 1>(s_v, lb, sc, vref, S, M); g2p_row<D, 2, 2>(s_v, lb, sc, vref, S, M);
  float* out = A.st_next;
#pragma unroll
  for (int a = 0; a < D; ++a) {
#pragma unroll
    for (int b = 0; b < D; ++b) Cn[a][b] = 4.f * P.fres * fmaf(-S[a], sc.fx[b], M[a][b]);
#pragma unroll
    for (int b = 0; b < D; ++b) {
      // F' = (I + dt C') F  <=>  H' = H + dt C' (I + H)  (Eq. 9 on H = F - I)
      float acc = fmaf(P.dt, Cn[a][b], H[a][b]);
#pragma unroll
      for (int c = 0; c < D; ++c) acc = fmaf(P.dt * Cn[a][c], H[c][b], acc);
      Hn[a][b] = acc;
      out[rix<D>(comp_F<D>(a, b), k, NT)] = acc;
      out[rix<D>(comp_C<D>(a, b), k, NT)] = Cn[a][b];
    }
    vn[a] = S[a] + (&vref.x)[a];
    out[rix<D>(comp_v<D>(a), k, NT)] = vn[a];
    x[a] = fmaf(P.dt, vn[a], x[a]);
    out[rix<D>(comp_x<D>(a), k, NT)] = x[a];
  }
  A.orig_next[k] = u;
  int gbn, key;
  const int e = key_of<D>(x, r, P, gbn, key);
  if (e) latch(A.err, e, A.t + 1, u);
  A.key_next[k] = key;
  // block histogram of step t+1 (threads of a warp mostly share one block)
  const unsigned am = __activemask();
  const unsigned peers = __match_any_sync(am, gbn);
  if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&A.cnt[gbn], __popc(peers));
  return e == E_OK;
}

template <int D, bool SPLIT = false>
__global__ __launch_bounds__(kThreads, MPM_G2P_MINB) void k_g2p(KParams P, StepArgs A) {
  MPM_PDL_ENTRY();
  __shared__ float4 s_v[Dim<D>::TN];
  __shared__ WorkSh<D> s_w;
  const size_t NT = P.NT;
  const int n_occ = A.info_t[I_NOCC];
  const int parts = work_parts<SPLIT>(n_occ);
  for (;;) {
    if (threadIdx.x == 0) claim_item<D, SPLIT>(P, A, I_WORK3, n_occ, parts, s_w);
    __syncthreads();
    const int n = s_w.n;
    if (n < 0) break;
    if (SPLIT && n == 0) {  // uniform; every thread has read s_w before thread 0 claims again
      __syncthreads();
      continue;
    }
    const int s = s_w.s, r = s_w.r;
    int bc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) bc[a] = s_w.bc[a];
    float4 vref, aref_unused;
#if MPM_G2P_PF
    for (int i = threadIdx.x; i < n; i += kThreads) {  // this block's x, F -> L2
      const int j = __ldg(&A.perm[s + i]);
      prefetch_record<D>(A.st, NT, j, 0, D);
      prefetch_record<D>(A.st, NT, j, comp_F<D>(0, 0), D * D);
    }
#endif
    stage_tile<D, false>(P, A, r, bc, s_v, nullptr, 0, vref, aref_unused);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kThreads) {
      float x[D], vn[D], Cn[D][D], Hn[D][D];
      int u;
      g2p_particle<D>(P, A, s_v, vref, bc, r, s + i, x, vn, Cn, Hn, u);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------
// Fused G2P2G (NEXT N2): one pass over the particles per step.  CTA per occupied
// block of step t: [SORT: the in-block cell sort of step t (perm)] -> stage grid t (fused grid
// update) -> G2P of each particle (state t+1 written to the tape) -> [SCAT: with the new
// state still in registers, the step-(t+1) stress and P2G payload -> in-CTA counting sort by
// the new cell -> the tile consumer -> RED flush into grid t+1].  Grid t+1's slot map is the
// dilated one (k_scan_lookback<D, true>): a particle whose new base cell left its block (a
// few per block) adds its 3^D nodes with direct vector REDs instead of through the tile.
// The (p, m) accumulated are those of the unfused P2G of step t+1 up to fp32 summation order.
// Saves the P2G re-read of the state (x, v, C, F, 96 B) and one launch per step.
// ------------------------------------------------------------------------------------
constexpr int kCapF = MPM_FUSE_CAP;  // particles per chunk of the fused kernel (payload buffer)
static_assert(kCapF % 256 == 0 && kCapF <= kCap, "pay_slot permutes aligned groups of 8 within the chunk");
template <int D>
constexpr int fuse_dyn_smem() {  // payload buffer; also holds the in-block sort (kSortCap ints)
  return (PayOf<D, false, MPM_FUSE_FX>::T::N * kCapF > kSortCap ? PayOf<D, false, MPM_FUSE_FX>::T::N * kCapF : kSortCap) *
         (int)sizeof(float);
}
// escapee code: the new base cell relative to the block, lb in [-EO, EO) per axis, EB bits
// each (EO > Bb, so a neighbour block's cells fit; D * EB <= 14 keeps -2 - code in a short)
template <int D> struct Esc { static constexpr int EB = D == 3 ? 4 : 5, EO = 1 << (EB - 1); };
static_assert(Esc<3>::EO > Dim<3>::BB && Esc<2>::EO > Dim<2>::BB, "escapee code range");
static_assert(3 * Esc<3>::EB <= 14 && 2 * Esc<2>::EB <= 14, "escapee code fits a short");

// the escapees' nodes (NS per escapee, one (escapee, node) pair per thread of the idle group
// [0, nthr)) as direct vector REDs into grid t+1; node value w_o (A + B o), mass w_o m from the
// escapee's payload slot
template <int D, int CAP = kCap, bool FX = false>
__device__ __forceinline__ void scatter_escapees(const KParams& P, const StepArgs& A, int r, const int* bc,
                                                 const float (*s_pay)[CAP], const short* s_cell,
                                                 const short* s_ord, int nesc, int it, int nthr) {
  using DD = Dim<D>;
  using PY = typename PayOf<D, false, FX>::T;
  constexpr int EB = Esc<D>::EB, EO = Esc<D>::EO;
  for (int idx = it; idx < nesc * DD::NS; idx += nthr) {
    const int e = idx / DD::NS;
    int q = idx - e * DD::NS;
    const int pi = s_ord[CAP - 1 - e];
    const int pk = -2 - (int)s_cell[pi];
    const int ps = pay_slot(pi);
    MPM_CHECK(ps >= 0 && ps < CAP);
    int o[D], nb_[D], loc[D];
    float W = 1.f;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      o[a] = q % 3;
      q /= 3;
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int lb = ((pk >> (EB * (D - 1 - a))) & (2 * EO - 1)) - EO;
      const int node = bc[a] * DD::BB + lb + o[a];
      W *= FX ? bspl(s_pay[PY::W + a][ps], o[a]) : s_pay[PY::W + a * 3 + o[a]][ps];
      nb_[a] = node >> DD::LOG_BB;
      loc[a] = node & (DD::BB - 1);
    }
    const int slot = __ldg(&A.slot_next[r * P.nb + block_lin<D>(nb_, P.nbpa)]);
    if (slot < 0) {  // moved more than the dilation allows (|v| dt >= dx)
      latch(A.err, E_FUSE, A.t + 1, -1);
      continue;
    }
    float val[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int a = 0; a < D; ++a) {
      float acc = s_pay[PY::A + a][ps];
#pragma unroll
      for (int b = 0; b < D; ++b) acc = fmaf((float)o[b], s_pay[PY::B + a * D + b][ps], acc);
      val[a] = W * acc;
    }
    atomicAdd(A.grid + (size_t)slot * kCPB + cell_lin<D>(loc), make_float4(val[0], val[1], val[2], W * s_pay[PY::M][ps]));
  }
}

template <int D, int MAT, bool SORT, bool SCAT, bool SPLIT = false>
__global__ __launch_bounds__(kThreads, MPM_FUSE_MINB) void k_g2p2g(KParams P, StepArgs A) {
  MPM_PDL_ENTRY();
  using DD = Dim<D>;
  using PY = typename PayOf<D, false, MPM_FUSE_FX>::T;
  constexpr int BB = DD::BB, TN = DD::TN;
  constexpr int EB = Esc<D>::EB, EO = Esc<D>::EO;
  __shared__ int s_hist[kCPB];
  __shared__ int s_cstart[kCPB + 1];
  __shared__ int s_cursor[kCPB];
  __shared__ int s_sort_st[(SORT && !SCAT) ? kSortCap : 1];  // SCAT: the sort uses the payload area
  __shared__ float4 s_v[TN];
  __shared__ float4 s_tile[3][SCAT ? TN : 1];
  __shared__ short s_cell[SCAT ? kCapF : 1];
  __shared__ short s_ord[SCAT ? kCapF : 1];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  float (*s_pay)[kCapF] = reinterpret_cast<float (*)[kCapF]>(s_dyn);  // [PY::N][kCapF], dynamic (SCAT)
  int* s_sort = SCAT ? reinterpret_cast<int*>(s_dyn) : s_sort_st;  // the sort is done before the payload is written
  __shared__ WorkSh<D> s_w;
  __shared__ int s_nesc;
  __shared__ int s_perm[MPM_FUSE_SPERM && SORT ? kCapPerm : 1];  // the sorted order of the block (SORT)
  const int tid = threadIdx.x;
  const int n_occ = A.info_t[I_NOCC];
  const int ox = tid / kCPB;
  const int c = D == 3 ? ((((tid >> 2) & 3) * 4 + ((tid >> 4) & 3)) * 4 + (tid & 3)) : tid % kCPB;
  // SPLIT (small problems, fewer occupied blocks than CTAs): a block's particles are shared by
  // up to 8 CTAs; each sorts the whole block (identical perm values; a block beyond kSortCap,
  // whose sort needs the global scratch, goes to its first part alone) and runs G2P and the
  // step-(t+1) scatter on its range of the sorted order, flushing a partial tile with REDs
  const int parts = work_parts<SPLIT>(n_occ);
  for (;;) {
    if (tid == 0) claim_item<D, SPLIT>(P, A, I_WORK3, n_occ, parts, s_w);
    __syncthreads();
    int n = s_w.n, s = s_w.s;
    if (n < 0) break;
    const int s0 = s_w.s0, n0 = s_w.n0;
    if (SPLIT && n0 > kSortCap) {  // uniform: the whole block to the part that starts it
      n = s == s0 ? n0 : 0;
      s = s0;
    }
    if (SPLIT && n == 0) {  // uniform; every thread has read s_w before thread 0 claims again
      __syncthreads();
      continue;
    }
    const int r = s_w.r;
    int bc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) bc[a] = s_w.bc[a];
    int myslot = -1;  // grid t+1 slots of the tile's blocks bc + {0, 1}^D (flush)
    if (SCAT) {
      const int lane = tid & 31;
      if (lane < (1 << D)) {
        int nb_[D];
        bool inside = true;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          nb_[a] = bc[a] + ((lane >> (D - 1 - a)) & 1);
          inside &= nb_[a] < P.nbpa;
        }
        if (inside) myslot = __ldg(&A.slot_next[r * P.nb + block_lin<D>(nb_, P.nbpa)]);
      }
      for (int i = tid; i < 3 * TN; i += kThreads) (&s_tile[0][0])[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float4 vref, aref_unused;
#if MPM_FUSE_STAGE_FIRST
    // grid t's tile first: its loads are independent of the sort and overlap its phases
    stage_tile<D, false>(P, A, r, bc, s_v, nullptr, 0, vref, aref_unused);
#endif
    bool pcrowd = true;
    if (SORT) {
      if (tid < kCPB) s_hist[tid] = 0;
      __syncthreads();
      pcrowd = block_cell_sort<D, true>(P, A, s0, n0, tid, s_hist, s_cstart, s_cursor, s_sort,
                                        MPM_FUSE_SPERM ? s_perm : nullptr);
    }
#if !MPM_FUSE_STAGE_FIRST
    stage_tile<D, false>(P, A, r, bc, s_v, nullptr, 0, vref, aref_unused);
#endif
    __syncthreads();
    for (int lo = 0; lo < n; lo += kCapF) {
      const int hi = min(n, lo + kCapF);
      if (SCAT) {
        if (tid < kCPB) s_hist[tid] = 0;
        if (tid == 0) s_nesc = 0;
        __syncthreads();
      }
      for (int pi = tid; pi < hi - lo; pi += kThreads) {
        float x[D], vn[D], Cn[D][D], Hn[D][D];
        int u, ai = -1;
        float4 pr;  // m, V, mu, lam
        // the sorted storage index from the sort's shared copy (no global round trip)
        const int pj = s + lo + pi - s0;  // position in the whole block's sorted order
        const int jin = (MPM_FUSE_SPERM && SORT && !pcrowd && pj < kCapPerm) ? s_perm[pj] : -1;
        const bool ok = g2p_particle<D, SORT, SCAT>(P, A, s_v, vref, bc, r, s + lo + pi, x, vn, Cn, Hn, u, &pr, &ai, jin);
        if constexpr (SCAT) {
          Stencil<D> sc;
          make_stencil<D>(x, P.fres, sc);
          int lb[D];
          bool inb = true;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            lb[a] = sc.base[a] - bc[a] * BB;
            inb &= (lb[a] >= 0) & (lb[a] < BB);
          }
          float Av[D], Bm[D][D];
          p2g_payload<D, MAT>(P, A, r, A.t + 1, u, pr, ai, vn, Hn, Cn, sc.fx, Av, Bm);
          int cell = -1;
          if (ok) {
            const int ps = pay_slot(pi);
            MPM_CHECK(ps >= 0 && ps < kCapF);
#pragma unroll
            for (int a = 0; a < D; ++a) {
              if (MPM_FUSE_FX) {
                s_pay[PY::W + a][ps] = sc.fx[a];
              } else {
#pragma unroll
                for (int o = 0; o < 3; ++o) s_pay[PY::W + a * 3 + o][ps] = sc.w[a][o];
              }
            }
            s_pay[PY::M][ps] = pr.x;
#pragma unroll
            for (int a = 0; a < D; ++a) {
              s_pay[PY::A + a][ps] = Av[a];
#pragma unroll
              for (int b = 0; b < D; ++b) s_pay[PY::B + a * D + b][ps] = Bm[a][b];
            }
            if (inb) {
              cell = cell_lin<D>(lb);
              atomicAdd(&s_hist[cell], 1);
            } else {
              // escapee (new base cell outside the block; CFL keeps it within a few cells):
              // its nodes go out as direct REDs after the sort, by the threads the consumer
              // leaves idle.  Code -2 - packed (lb + EO, EB bits per axis); its index is kept
              // at the top of s_ord (the block's own particles fill it from the bottom).
              int pk = 0;
              bool near = true;
#pragma unroll
              for (int a = 0; a < D; ++a) {
                near &= (lb[a] >= -EO) & (lb[a] < EO);
                pk = (pk << EB) | ((lb[a] + EO) & (2 * EO - 1));
              }
              if (near) {
                cell = -2 - pk;
                s_ord[kCapF - 1 - atomicAdd(&s_nesc, 1)] = (short)pi;
              } else {
                latch(A.err, E_FUSE, A.t + 1, u);
              }
            }
          }
          s_cell[pi] = (short)cell;
        }
      }
      if constexpr (SCAT) {
        __syncthreads();
        cell_scan(s_hist, s_cstart, s_cursor, tid);
        __syncthreads();
        for (int pi = tid; pi < hi - lo; pi += kThreads) {
          const int cl = s_cell[pi];
          if (cl >= 0) {
            const int at = atomicAdd(&s_cursor[cl], 1);
            MPM_CHECK(at >= 0 && at < kCapF - s_nesc);
            s_ord[at] = (short)pi;
          }
        }
        __syncthreads();
        const int i0 = tid < 3 * kCPB ? s_cstart[c] : 0;
        const int i1 = tid < 3 * kCPB ? s_cstart[c + 1] : 0;
        scatter_consume<D, false, true, kCapF, MPM_FUSE_FX>(s_pay, s_tile, i0, i1, s_ord, ox, c, tid);
        if (tid >= 3 * kCPB)
          scatter_escapees<D, kCapF, MPM_FUSE_FX>(P, A, r, bc, s_pay, s_cell, s_ord, s_nesc, tid - 3 * kCPB,
                                                  kThreads - 3 * kCPB);
        __syncthreads();
      }
    }
    if constexpr (SCAT) scatter_flush<D, false>(P, A.grid, s_tile, bc, myslot, 0, tid);
    __syncthreads();
  }
}

// ---- P2G^T gather (steps F-K and J; E/nu per R19) in the Kirchhoff form:
//   T = dL/dtau = -k Q, Q = dL/dG = sum_i w dp_i (x_i - x_p)^T, k = 4 dt V / dx^2
//   dv^t = m sum_i w dp_i ; dC^t = m Q
//   dF^t = (I + dt C^{t+1})^T dF^{t+1} + mu (T + T^T) F + lam tr(T) F^{-T} + (T + T^T) F sigma
//   dx^t = dx^{t+1} + sum_i dW_i s_i - 4 res^2 g_C^T v^{t+1} - G^T sum_i w dp_i
//     s_i = v_i . u(o) + dp_i . q(o) + m dm_i,  u(o) = g_v + 4 res g_C (o - fx)  (the G2P^T
//     payload), q(o) = m v + dx G (o - fx) (the P2G payload) -- both affine in o
//   dsigma = F^T T F (diag -> actuation); dmu = T : (F F^T - I); dlam = tr(T) ln J
// Two passes over the 3^D stencil keep the live set small: the v-pass (S, M_v, sum dW v.u)
// and the dp-pass (S_d, M_d, sum dW (dp.q + m dm)).
// Per (ox, oy) row the oz-sums sum wz f and sum oz wz f are formed, then folded.
template <int D> struct PassAcc {
  float S[D];      // sum W f_i
  float M[D][D];   // sum W f_i o_b
  float g[D];      // sum dW (f_i . c(o) + e_i)
  float Se;        // sum W (.w)   (dp-pass only: sum W dL/dm_i, for the mass gradient)
};

// one pass; F4 = tile of float4 (f = .xyz, e = em * .w), c(o) = c0 + Cm o
template <int D, int OX, int OY, bool WS, bool EM = true>
__device__ __forceinline__ void pass_row(const float4* tile, const int* lb, const float (&w)[D][3],
                                         const float (&dw)[D][3], const float* c0, const float (&Cm)[D][D],
                                         float em, const float4& ref, PassAcc<D>& R) {
  float cxy[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    cxy[a] = c0[a];
    if (OX) cxy[a] = fmaf((float)OX, Cm[a][0], cxy[a]);
    if (OY) cxy[a] = fmaf((float)OY, Cm[a][1], cxy[a]);
  }
  float A0[D], A1[D], t1 = 0.f, t2 = 0.f, Aw = 0.f;
#pragma unroll
  for (int a = 0; a < D; ++a) A0[a] = A1[a] = 0.f;
  if constexpr (D == 3) {
#pragma unroll
    for (int oz = 0; oz < 3; ++oz) {
      const float4 q = tile[tile_idx<D, OX, OY, 0>(lb) + oz];
      const float f[3] = {q.x - ref.x, q.y - ref.y, q.z - ref.z};
      float sv = EM ? em * (q.w - ref.w) : 0.f;  // EM = false: no e_i term (v-pass; 0 * q.w is not foldable)
#pragma unroll
      for (int a = 0; a < 3; ++a) sv = fmaf(f[a], oz == 0 ? cxy[a] : fmaf((float)oz, Cm[a][2], cxy[a]), sv);
      const float wz = w[2][oz];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        A0[a] = fmaf(wz, f[a], A0[a]);
        if (oz) A1[a] = fmaf((float)oz * wz, f[a], A1[a]);
      }
      t1 = fmaf(wz, sv, t1);
      t2 = fmaf(dw[2][oz], sv, t2);
      if (WS) Aw = fmaf(wz, q.w - ref.w, Aw);
    }
    const float wx = w[0][OX], wy = w[1][OY], wxy = wx * wy;
    if (WS) R.Se = fmaf(wxy, Aw, R.Se);
    R.g[0] = fmaf(dw[0][OX] * wy, t1, R.g[0]);
    R.g[1] = fmaf(wx * dw[1][OY], t1, R.g[1]);
    R.g[2] = fmaf(wxy, t2, R.g[2]);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      R.S[a] = fmaf(wxy, A0[a], R.S[a]);
      if (OX) R.M[a][0] = fmaf((float)OX * wxy, A0[a], R.M[a][0]);
      if (OY) R.M[a][1] = fmaf((float)OY * wxy, A0[a], R.M[a][1]);
      R.M[a][2] = fmaf(wxy, A1[a], R.M[a][2]);
    }
  } else {
    const float4 q = tile[tile_idx<D, OX, OY, 0>(lb)];
    const float f[2] = {q.x - ref.x, q.y - ref.y};
    float sv = EM ? em * (q.w - ref.w) : 0.f;
#pragma unroll
    for (int a = 0; a < 2; ++a) sv = fmaf(f[a], cxy[a], sv);
    const float wx = w[0][OX], wy = w[1][OY], wxy = wx * wy;
    if (WS) R.Se = fmaf(wxy, q.w - ref.w, R.Se);
    R.g[0] = fmaf(dw[0][OX] * wy, sv, R.g[0]);
    R.g[1] = fmaf(wx * dw[1][OY], sv, R.g[1]);
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      R.S[a] = fmaf(wxy, f[a], R.S[a]);
      if (OX) R.M[a][0] = fmaf((float)OX * wxy, f[a], R.M[a][0]);
      if (OY) R.M[a][1] = fmaf((float)OY * wxy, f[a], R.M[a][1]);
    }
  }
}

// 3-D pass with packed fp32x2 FMAs (sm_100 FFMA2): the (x, y) components of S, M and the
// (g0, g1) / (t1, t2) pairs advance in one instruction; per component the same fused op as fmaf
struct PassAcc2 {
  float2 S, M0, M1, M2, g01;  // (x, y) of S, M[.][0..2], (g0, g1)
  float Sz, Mz0, Mz1, Mz2, g2, Se;
};

template <int OX, int OY, bool WS>
__device__ __forceinline__ void pass_row2(const float4* tile, const int* lb, const float (&w)[3][3],
                                          const float (&dw)[3][3], const float* c0, const float (&Cm)[3][3],
                                          float em, PassAcc2& R) {
  float cxy[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    cxy[a] = c0[a];
    if (OX) cxy[a] = fmaf((float)OX, Cm[a][0], cxy[a]);
    if (OY) cxy[a] = fmaf((float)OY, Cm[a][1], cxy[a]);
  }
  float2 A0 = make_float2(0.f, 0.f), A1 = A0, t12 = A0;
  float A0z = 0.f, A1z = 0.f, Aw = 0.f;
#pragma unroll
  for (int oz = 0; oz < 3; ++oz) {
    const float4 q = tile[tile_idx<3, OX, OY, 0>(lb) + oz];
    float sv = em * q.w;
#pragma unroll
    for (int a = 0; a < 3; ++a) sv = fmaf((&q.x)[a], oz == 0 ? cxy[a] : fmaf((float)oz, Cm[a][2], cxy[a]), sv);
    const float wz = w[2][oz];
    const float2 fxy = make_float2(q.x, q.y);
    A0 = __ffma2_rn(make_float2(wz, wz), fxy, A0);
    A0z = fmaf(wz, q.z, A0z);
    if (oz) {
      const float ow = (float)oz * wz;
      A1 = __ffma2_rn(make_float2(ow, ow), fxy, A1);
      A1z = fmaf(ow, q.z, A1z);
    }
    t12 = __ffma2_rn(make_float2(wz, dw[2][oz]), make_float2(sv, sv), t12);
    if (WS) Aw = fmaf(wz, q.w, Aw);
  }
  const float wx = w[0][OX], wy = w[1][OY], wxy = wx * wy;
  if (WS) R.Se = fmaf(wxy, Aw, R.Se);
  const float2 gw = __fmul2_rn(make_float2(dw[0][OX], wx), make_float2(wy, dw[1][OY]));
  R.g01 = __ffma2_rn(gw, make_float2(t12.x, t12.x), R.g01);
  R.g2 = fmaf(wxy, t12.y, R.g2);
  const float2 w2 = make_float2(wxy, wxy);
  R.S = __ffma2_rn(w2, A0, R.S);
  R.Sz = fmaf(wxy, A0z, R.Sz);
  if (OX) {
    const float v = (float)OX * wxy;
    R.M0 = __ffma2_rn(make_float2(v, v), A0, R.M0);
    R.Mz0 = fmaf(v, A0z, R.Mz0);
  }
  if (OY) {
    const float v = (float)OY * wxy;
    R.M1 = __ffma2_rn(make_float2(v, v), A0, R.M1);
    R.Mz1 = fmaf(v, A0z, R.Mz1);
  }
  R.M2 = __ffma2_rn(w2, A1, R.M2);
  R.Mz2 = fmaf(wxy, A1z, R.Mz2);
}

template <bool WS>
__device__ __forceinline__ void stencil_pass2(const float4* tile, const int* lb, const float (&w)[3][3],
                                              const float (&dw)[3][3], const float* c0, const float (&Cm)[3][3],
                                              float em, PassAcc<3>& Ro) {
  PassAcc2 R;
  R.S = R.M0 = R.M1 = R.M2 = R.g01 = make_float2(0.f, 0.f);
  R.Sz = R.Mz0 = R.Mz1 = R.Mz2 = R.g2 = R.Se = 0.f;
  pass_row2<0, 0, WS>(tile, lb, w, dw, c0, Cm, em, R); pass_row2<0, 1, WS>(tile, lb, w, dw, c0, Cm, em, R);
  pass_row2<0, 2, WS>(tile, lb, w, dw, c0, Cm, em, R); pass_row2<1, 0, WS>(tile, lb, w, dw, c0, Cm, em, R);
  pass_row2<1, 1, WS>(tile, lb, w, dw, c0, Cm, em, R); pass_row2<1, 2, WS>(tile, lb, w, dw, c0, Cm, em, R);
  pass_row2<2, 0, WS>(tile, lb, w, dw, c0, Cm, em, R); pass_row2<2, 1, WS>(tile, lb, w, dw, c0, Cm, em, R);
  pass_row2<2, 2, WS>(tile, lb, w, dw, c0, Cm, em, R);
  Ro.S[0] = R.S.x; Ro.S[1] = R.S.y; Ro.S[2] = R.Sz;
  Ro.M[0][0] = R.M0.x; Ro.M[1][0] = R.M0.y; Ro.M[2][0] = R.Mz0;
  Ro.M[0][1] = R.M1.x; Ro.M[1][1] = R.M1.y; Ro.M[2][1] = R.Mz1;
  Ro.M[0][2] = R.M2.x; Ro.M[1][2] = R.M2.y; Ro.M[2][2] = R.Mz2;
  Ro.g[0] = R.g01.x; Ro.g[1] = R.g01.y; Ro.g[2] = R.g2;
  Ro.Se = R.Se;
}

template <int D, bool WS, bool F2 = false, bool EM = true>
__device__ __forceinline__ void stencil_pass(const float4* tile, const int* lb, const float (&w)[D][3],
                                             const float (&dw)[D][3], const float* c0,
                                             const float (&Cm)[D][D], float em, const float4& ref,
                                             PassAcc<D>& R) {
#pragma unroll
  for (int a = 0; a < D; ++a) {
    R.S[a] = R.g[a] = 0.f;
#pragma unroll
    for (int b = 0; b < D; ++b) R.M[a][b] = 0.f;
  }
  R.Se = 0.f;
  if constexpr (D == 3 && F2) {
    stencil_pass2<WS>(tile, lb, w, dw, c0, Cm, em, R);  // ref is zero at every call site
    return;
  }
  pass_row<D, 0, 0, WS, EM>(tile, lb, w, dw, c0, Cm, em, ref, R); pass_row<D, 0, 1, WS, EM>(tile, lb, w, dw, c0, Cm, em, ref, R);
  pass_row<D, 0, 2, WS, EM>(tile, lb, w, dw, c0, Cm, em, ref, R); pass_row<D, 1, 0, WS, EM>(tile, lb, w, dw, c0, Cm, em, ref, R);
  pass_row<D, 1, 1, WS, EM>(tile, lb, w, dw, c0, Cm, em, ref, R); pass_row<D, 1, 2, WS, EM>(tile, lb, w, dw, c0, Cm, em, ref, R);
  pass_row<D, 2, 0, WS, EM>(tile, lb, w, dw, c0, Cm, em, ref, R); pass_row<D, 2, 1, WS, EM>(tile, lb, w, dw, c0, Cm, em, ref, R);
  pass_row<D, 2, 2, WS, EM>(tile, lb, w, dw, c0, Cm, em, ref, R);
}

// P2G^T's shared-memory park of one particle (rows of MPM_P2GT_THREADS floats): incoming
// dL/dx, dL/dF; the state's H; v; C
template <int D> constexpr int kParkH = D + D * D;
template <int D> constexpr int kParkV = kParkH<D> + D * D;
template <int D> constexpr int kParkC = kParkV<D> + D;
template <int D> constexpr int kParkN = MPM_P2GT_PARK >= 3 ? kParkC<D> + D * D : MPM_P2GT_PARK >= 2 ? kParkV<D> : MPM_P2GT_PARK ? kParkH<D> : 1;
template <int D>
__device__ __forceinline__ void park_H(const StepArgs& A, size_t NT, int j, const float* park, float (&H)[D][D]) {
#if MPM_P2GT_PARK >= 2
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) H[a][b] = park[(kParkH<D> + a * D + b) * MPM_P2GT_THREADS];
#else
  load_H<D>(A.st, NT, j, H);
#endif
}

template <int D, bool MG, int MAT>
__device__ __forceinline__ void p2g_adj_particle(const KParams& P, const StepArgs& A, const float4* s_v,
                                                 const float4* s_a, const float4& aref, const int* bc,
                                                 int r, int k, int& aid_out, float* dsig_out, float* park,
                                                 int j_in = -1, int u_in = -1) {
  const size_t NT = P.NT;
  const float* gi = A.gin;
  // (j, u) from the caller's shared copy of the item's perm / orig (MPM_P2GT_IDXSM), else loaded
  const int j = j_in >= 0 ? j_in : __ldg(&A.perm[k]);
  const int u = u_in >= 0 ? u_in : __ldg(&A.orig_next[k]);  // = orig_t[perm[k]] (written by G2P of this step)
  const float4 pr = __ldg(&A.prm[u]);
  const int ai = __ldg(&A.aid[u]);
  const float dmu0 = A.dmu[u], dlam0 = A.dlam[u];  // accumulators: loaded early, stored at the end
  const float dm0 = MG ? A.dmass[u] : 0.f;
  const float kk = 4.f * P.fres * P.fres * P.dt * pr.y;
#if MPM_P2GT_SIG_EARLY
  // the actuation of this particle (third load of the chain orig -> aid -> act), issued before
  // the v-pass so that its latency overlaps the pass
  float sig[D];
#pragma unroll
  for (int a = 0; a < D; ++a)
    sig[a] = ai >= 0 ? P.act_s * __ldg(&A.act[(((size_t)r * P.T + A.t) * P.K + ai) * D + a]) : 0.f;
#endif
  float x[D];
#pragma unroll
  for (int a = 0; a < D; ++a) x[a] = __ldg(&A.st[rix<D>(comp_x<D>(a), j, NT)]);
  Stencil<D> sc;
  make_stencil<D>(x, P.fres, sc);
  float dw[D][3];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    stencil_dw(sc.fx[a], dw[a]);
#pragma unroll
    for (int o = 0; o < 3; ++o) dw[a][o] *= P.fres;
  }
  int lb[D];
#pragma unroll
  for (int a = 0; a < D; ++a) lb[a] = sc.base[a] - bc[a] * Dim<D>::BB;

  // ---- v-pass: c(o) = u(o) = g_v + 4 res g_C (o - fx)   (steps A, B) ----
  PassAcc<D> Rv;
  float Cn[D][D];  // C^{t+1} (Eq. 8 recomputed)
  float gxv[D];
  {
    float u0[D], U[D][D];
#if MPM_P2GT_PARK
    // the incoming dL/dx and dL/dF of this particle, parked in shared memory for the epilogue
    // ((J), (H)) instead of re-read from global memory there (a stride of the CTA size:
    // conflict-free)
#pragma unroll
    for (int a = 0; a < D; ++a) {
      park[a * MPM_P2GT_THREADS] = gi[rix<D>(comp_x<D>(a), k, NT)];
#pragma unroll
      for (int b = 0; b < D; ++b) park[(D + a * D + b) * MPM_P2GT_THREADS] = gi[rix<D>(comp_F<D>(a, b), k, NT)];
    }
#endif
#if MPM_P2GT_PARK >= 2  // and the state's H (read by the stress and by (H), (K))
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b)
        park[(kParkH<D> + a * D + b) * MPM_P2GT_THREADS] = __ldg(&A.st[rix<D>(comp_F<D>(a, b), j, NT)]);
#endif
#if MPM_P2GT_PARK >= 3  // and the state's v, C (the dp-pass payload)
#pragma unroll
    for (int a = 0; a < D; ++a) {
      park[(kParkV<D> + a) * MPM_P2GT_THREADS] = __ldg(&A.st[rix<D>(comp_v<D>(a), j, NT)]);
#pragma unroll
      for (int b = 0; b < D; ++b)
        park[(kParkC<D> + a * D + b) * MPM_P2GT_THREADS] = __ldg(&A.st[rix<D>(comp_C<D>(a, b), j, NT)]);
    }
#endif
#pragma unroll
    for (int a = 0; a < D; ++a) {
      u0[a] = fmaf(P.dt, gi[rix<D>(comp_x<D>(a), k, NT)], gi[rix<D>(comp_v<D>(a), k, NT)]);
#pragma unroll
      for (int b = 0; b < D; ++b) {
        // g_C = gC + dt gF F^T with F = I + H
        float gc = fmaf(P.dt, gi[rix<D>(comp_F<D>(a, b), k, NT)], gi[rix<D>(comp_C<D>(a, b), k, NT)]);
#pragma unroll
        for (int c = 0; c < D; ++c)
          gc = fmaf(P.dt * gi[rix<D>(comp_F<D>(a, c), k, NT)], __ldg(&A.st[rix<D>(comp_F<D>(b, c), j, NT)]), gc);
        U[a][b] = 4.f * P.fres * gc;
        u0[a] = fmaf(-U[a][b], sc.fx[b], u0[a]);
      }
    }
    stencil_pass<D, false, (MPM_FFMA2_P2GT & 1) != 0, false>(s_v, lb, sc.w, dw, u0, U, 0.f, make_float4(0.f, 0.f, 0.f, 0.f), Rv);
    // dx term -4 res^2 g_C^T v^{t+1} = -res U^T S_v
#pragma unroll
    for (int a = 0; a < D; ++a) {
      float acc = Rv.g[a];
#pragma unroll
      for (int b = 0; b < D; ++b) acc = fmaf(-P.fres * U[b][a], Rv.S[b], acc);
      gxv[a] = acc;
#pragma unroll
      for (int b = 0; b < D; ++b) Cn[a][b] = 4.f * P.fres * fmaf(-Rv.S[a], sc.fx[b], Rv.M[a][b]);
    }
  }
  // ---- dp-pass: c(o) = q(o) = m v + dx G (o - fx), e_i = m dm_i   (Eqs. 4-5) ----
#if !MPM_P2GT_SIG_EARLY
  float sig[D];
#pragma unroll
  for (int a = 0; a < D; ++a)
    sig[a] = ai >= 0 ? P.act_s * __ldg(&A.act[(((size_t)r * P.T + A.t) * P.K + ai) * D + a]) : 0.f;
#endif
  PassAcc<D> Rd;
  float Gm[D][D];  // dx G
  {
    float H[D][D], tau[D][D], q0[D];
    park_H<D>(A, NT, j, park, H);
    if constexpr (MAT == 1) kirchhoff_fcr<D>(H, pr.z, pr.w, sig, tau, det1m<D>(H));
    else kirchhoff_h<D>(H, pr.z, pr.w, sig, tau, log1pf(det1m<D>(H)));
#pragma unroll
    for (int a = 0; a < D; ++a) {
      q0[a] = pr.x * (MPM_P2GT_PARK >= 3 ? park[(kParkV<D> + a) * MPM_P2GT_THREADS] : __ldg(&A.st[rix<D>(comp_v<D>(a), j, NT)]));
#pragma unroll
      for (int b = 0; b < D; ++b) {
        Gm[a][b] = P.dx * fmaf(-kk, tau[a][b],
                               pr.x * (MPM_P2GT_PARK >= 3 ? park[(kParkC<D> + a * D + b) * MPM_P2GT_THREADS]
                                                          : __ldg(&A.st[rix<D>(comp_C<D>(a, b), j, NT)])));
        q0[a] = fmaf(-Gm[a][b], sc.fx[b], q0[a]);
      }
    }
    stencil_pass<D, MG, (MPM_FFMA2_P2GT & 2) != 0>(s_a, lb, sc.w, dw, q0, Gm, pr.x, make_float4(0.f, 0.f, 0.f, 0.f), Rd);
  }
  const float m = pr.x;
  float* go = A.gout;
  float Q[D][D], T[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
#pragma unroll
    for (int b = 0; b < D; ++b) {
      Q[a][b] = P.dx * fmaf(-Rd.S[a], sc.fx[b], Rd.M[a][b]);
      T[a][b] = -kk * Q[a][b];
      go[rix<D>(comp_C<D>(a, b), j, NT)] = m * Q[a][b];  // (I)
    }
    go[rix<D>(comp_v<D>(a), j, NT)] = m * (Rd.S[a] + (&aref.x)[a]);  // (F): sum W dp = S' + dp_ref
  }
  // (J): dx = gx + sum dW s - 4res^2 g_C^T S_v - G^T S_d
#pragma unroll
  for (int a = 0; a < D; ++a) {
    float acc = (MPM_P2GT_PARK ? park[a * MPM_P2GT_THREADS] : gi[rix<D>(comp_x<D>(a), k, NT)]) + gxv[a] + Rd.g[a];
#pragma unroll
    for (int b = 0; b < D; ++b) acc = fmaf(-P.fres * Gm[b][a], Rd.S[b], acc);
    go[rix<D>(comp_x<D>(a), j, NT)] = acc;
  }
  // (H), (K), material parameters
  float H[D][D], F[D][D];
  park_H<D>(A, NT, j, park, H);
  F_of_H<D>(H, F);
  const float jm1 = det1m<D>(H);
  const float J = 1.f + jm1;
  const float lnJ = log1pf(jm1);
  float FiT[D][D];
  inv_T<D>(F, J, FiT);
  float trT = 0.f;
#pragma unroll
  for (int a = 0; a < D; ++a) trT += T[a][a];
  // fixed-corotated (R21): tau_el = 2 mu (B - V) + lam J (J - 1) I.  With Y solving
  // V Y + Y V = sym(T) (diagonal in V's eigenbasis: Y' = (Q^T sym(T) Q) / (s_i + s_j)),
  // dL/dF = 2 mu ((T + T^T) F - 2 Y F) + lam (2J - 1) J tr(T) F^-T;  dL/dmu = 2 T : (B - V)
  float YF[D][D] = {}, dmu_fcr = 0.f;
  if constexpr (MAT == 1) {
    Stretch<D> sv;
    left_stretch<D>(H, sv);
    float M[D][D], Y[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int q = 0; q < D; ++q) {
        float acc = 0.f;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b < D; ++b) acc = fmaf(sv.Q[a][i] * 0.5f * (T[a][b] + T[b][a]), sv.Q[b][q], acc);
        M[i][q] = acc;
      }
#pragma unroll
    for (int i = 0; i < D; ++i) dmu_fcr = fmaf(2.f * sv.g[i], M[i][i], dmu_fcr);
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
          for (int q = 0; q < D; ++q) acc = fmaf(sv.Q[a][i] * M[i][q] / (sv.s[i] + sv.s[q]), sv.Q[b][q], acc);
        Y[a][b] = acc;
      }
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) {
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < D; ++c) acc = fmaf(Y[a][c], F[c][b], acc);
        YF[a][b] = acc;
      }
  }
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      float acc = MPM_P2GT_PARK ? park[(D + a * D + b) * MPM_P2GT_THREADS] : gi[rix<D>(comp_F<D>(a, b), k, NT)];
      float tf = 0.f;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        acc = fmaf(P.dt * Cn[c][a],
                   MPM_P2GT_PARK ? park[(D + c * D + b) * MPM_P2GT_THREADS] : gi[rix<D>(comp_F<D>(c, b), k, NT)], acc);
        tf = fmaf(T[a][c] + T[c][a], F[c][b], tf);
      }
      if constexpr (MAT == 1) {
        acc = fmaf(2.f * pr.z + sig[b], tf, acc);  // 2 mu (T+T^T) F + (T+T^T) F sigma
        acc = fmaf(-4.f * pr.z, YF[a][b], acc);
        acc = fmaf(pr.w * (2.f * J - 1.f) * J * trT, FiT[a][b], acc);
      } else {
        acc = fmaf(pr.z + sig[b], tf, acc);  // mu (T+T^T) F + (T+T^T) F sigma
        acc = fmaf(pr.w * trT, FiT[a][b], acc);
      }
      go[rix<D>(comp_F<D>(a, b), j, NT)] = acc;
    }
  float dmu = 0.f;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    float ds = 0.f;
#pragma unroll
    for (int b = 0; b < D; ++b) {
      float tf = 0.f;
#pragma unroll
      for (int c = 0; c < D; ++c) tf = fmaf(T[b][c], F[c][a], tf);
      ds = fmaf(F[b][a], tf, ds);
      if constexpr (MAT == 0) dmu = fmaf(T[a][b], ffti<D>(H, a, b), dmu);  // T : (F F^T - I), formed from H
    }
    dsig_out[a] = P.act_s * ds;
  }
  if constexpr (MAT == 1) dmu = dmu_fcr;
  A.dmu[u] = dmu0 + dmu;  // plain RMW (unique per particle): measured 36 us faster than a fp32 RED
  if (MG) {
    // NEXT N3: dL/dm_p = sum_i W dm_i + v . sum_i W dp_i + C : Q  (chain rule through Eqs. 3-5;
    // m enters m_i, m v and the m C part of G)
    float gmass = Rd.Se + aref.w;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      gmass = fmaf(__ldg(&A.st[rix<D>(comp_v<D>(a), j, NT)]), Rd.S[a] + (&aref.x)[a], gmass);
#pragma unroll
      for (int b = 0; b < D; ++b) gmass = fmaf(__ldg(&A.st[rix<D>(comp_C<D>(a, b), j, NT)]), Q[a][b], gmass);
    }
    A.dmass[u] = dm0 + gmass;
  }
  A.dlam[u] = dlam0 + trT * (MAT == 1 ? J * jm1 : lnJ);  // dtau/dlam = J (J - 1) I (R21) | ln J I (R1)
  aid_out = ai;
}

// Segmented warp reduction of the actuation gradient (step K -> dL/da[r][t][k]): one
// butterfly sum per distinct actuator id in the warp, added by one lane into the warp's own
// shared-memory slot; the CTA sums its warps' slots and adds them to global memory once per
// rollout it worked on (one global RED per actuator component per CTA instead of per warp:
// every warp adding to the same K*D addresses serialised in L2).  Called by all 32 lanes
// (key < 0 = no contribution).
template <int D>
__device__ __forceinline__ void reduce_actuation(float* w_da, int key, const float* v) {
  const int lane = threadIdx.x & 31;
  unsigned todo = __ballot_sync(0xffffffffu, key >= 0);
  while (todo) {
    const int src = __ffs(todo) - 1;
    const int k0 = __shfl_sync(0xffffffffu, key, src);
    const bool mine = key == k0;
    todo &= ~__ballot_sync(0xffffffffu, mine);
#pragma unroll
    for (int a = 0; a < D; ++a) {
      float s = mine ? v[a] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == src) w_da[k0 * D + a] += s;  // this warp's slot: one lane per key, no atomics
    }
  }
}

template <int D, bool MG, int MAT = 0, bool SPLIT = false>
__global__ __launch_bounds__(MPM_P2GT_THREADS, MPM_P2GT_MINB) void k_p2g_adj(KParams P, StepArgs A) {
  MPM_PDL_ENTRY();
  constexpr int NW = MPM_P2GT_THREADS / 32;
  __shared__ float4 s_v[Dim<D>::TN];
  __shared__ float4 s_a[Dim<D>::TN];
#if MPM_P2GT_CLAIM
  __shared__ WorkSh<D> s_w;
#else
  __shared__ int s_blk;
#endif
  __shared__ float s_da[NW][kMaxAct * D];  // per-warp dL/da[r][t][:][:] partial sums
  __shared__ float s_park[kParkN<D> * MPM_P2GT_THREADS];  // p2g_adj_particle's parked record
#if MPM_P2GT_IDXSM
  __shared__ int s_pj[kIdxCap], s_pu[kIdxCap];  // the item's perm / orig (first kIdxCap particles)
#endif
  __shared__ int s_da_r;                   // the rollout they belong to (-1: none)
  const int n_occ = A.info_t[I_NOCC];
  const size_t abase = (size_t)A.info_t[I_BASE] * kCPB;
  [[maybe_unused]] const size_t NT = P.NT;  // used by the optional record prefetch (MPM_P2GT_PF)
  const int KD = P.K * D;
  for (int q = threadIdx.x; q < NW * kMaxAct * D; q += MPM_P2GT_THREADS) (&s_da[0][0])[q] = 0.f;
  if (threadIdx.x == 0) s_da_r = -1;
  auto flush_da = [&](int rr) {  // all threads, after a barrier: sum the warps' slots
    for (int q = threadIdx.x; q < KD; q += MPM_P2GT_THREADS) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        v += s_da[w][q];
        s_da[w][q] = 0.f;
      }
      if (v != 0.f) atomicAdd(&A.da[((size_t)rr * P.T + A.t) * KD + q], v);
    }
  };
  const int parts = work_parts<SPLIT>(n_occ);
  // small problems (SPLIT): gridT of this step runs in the tile staging (a launch fewer on a
  // latency-bound chain; at C4 scale it costs more inside the staging than the k_grid_adj launch
  // it saves: P2G^T +18 us for gridT's 10); its other job moves here: zero the adjoint grid of
  // step t-1 (G2P^T of t-1 accumulates into it) and reset that step's work counters
  constexpr bool RAW = (SPLIT || MPM_GRIDT_FUSED >= 2) && MPM_GRIDT_FUSED;
  if (RAW && A.info_prev) adj_prepare(A.info_prev, A.agrid_prev, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
  for (;;) {
#if MPM_P2GT_CLAIM
    if (threadIdx.x == 0) claim_item<D, SPLIT>(P, A, I_WORK4, n_occ, parts, s_w);
    __syncthreads();
    const int n = s_w.n;
    if (n < 0) break;
    if (SPLIT && n == 0) {  // uniform; every thread has read s_w before thread 0 claims again
      __syncthreads();
      continue;
    }
    const int s = s_w.s, r = s_w.r;
    int bc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) bc[a] = s_w.bc[a];
#else
    if (threadIdx.x == 0) s_blk = atomicAdd(&A.info_t[I_WORK4], 1);
    __syncthreads();
    int gb, s, n;
    if (!work_item<SPLIT>(P, A, s_blk, n_occ, parts, gb, s, n)) break;
    if (SPLIT && n == 0) {  // uniform; every thread has read s_blk before thread 0 claims again
      __syncthreads();
      continue;
    }
    int r, bc[D];
    block_coords<D>(P, gb, r, bc);
#endif
    if (KD > 0 && r != s_da_r) {  // uniform: a new rollout -> flush the previous one's sums
      if (s_da_r >= 0) flush_da(s_da_r);
      __syncthreads();
      if (threadIdx.x == 0) s_da_r = r;  // read again only after the next claim barrier
    }
    float4 vref, aref;  // block-centre shifts (see stage_tile)
#if MPM_P2GT_PF
    for (int i = threadIdx.x; i < n; i += MPM_P2GT_THREADS) {  // this block's particle records -> L2
      const int k = s + i, j = __ldg(&A.perm[k]), u = __ldg(&A.orig_next[k]);
      prefetch_record<D>(A.st, NT, j, 0, Dim<D>::S);
      prefetch_record<D>(A.gin, NT, k, 0, Dim<D>::S);
      prefetch_l2(&A.prm[u]);
    }
#endif
#if MPM_P2GT_IDXSM
    // the item's (perm, orig) entries, read coalesced into shared memory while the tile is
    // staged: a particle's record loads then wait on one global round trip instead of two
    for (int q = threadIdx.x; q < min(n, kIdxCap); q += MPM_P2GT_THREADS) {
      s_pj[q] = __ldg(&A.perm[s + q]);
      s_pu[q] = __ldg(&A.orig_next[s + q]);
    }
#endif
    stage_tile<D, true, MPM_P2GT_THREADS, RAW>(P, A, r, bc, s_v, s_a, abase, vref, aref);
    __syncthreads();
    for (int i0 = 0; i0 < n; i0 += MPM_P2GT_THREADS) {  // uniform trip count: whole warps reach the reduction
      const int i = i0 + threadIdx.x;
      int ai = -1;
      float dsig[D] = {};
#if MPM_P2GT_IDXSM
      if (i < n)
        p2g_adj_particle<D, MG, MAT>(P, A, s_v, s_a, aref, bc, r, s + i, ai, dsig, s_park + threadIdx.x,
                                     i < kIdxCap ? s_pj[i] : -1, i < kIdxCap ? s_pu[i] : -1);
#else
      if (i < n) p2g_adj_particle<D, MG, MAT>(P, A, s_v, s_a, aref, bc, r, s + i, ai, dsig, s_park + threadIdx.x);
#endif
      __syncwarp();
      if (P.K > 0) reduce_actuation<D>(s_da[threadIdx.x >> 5], ai, dsig);
    }
    __syncthreads();
  }
  if (KD > 0 && s_da_r >= 0) flush_da(s_da_r);
}

// ------------------------------------------------------------------------------------
// NEXT N1: closed-loop controller embedded in P2G (Fig. 2 caption P:84):
//   z_t = [target, CoM_k, V_k (k < K)] per rollout, CoM_k / V_k = mass-weighted means over the
//   particles of actuator group k (DESIGN R20);  a_t = tanh(W z_t + b) -> act[r][t][k][:].
// Reverse (chain rule, SPEC controller_adjoint): g_pre = dL/da_t * (1 - a_t^2), dL/dz = W^T g_pre
// into dL/dx_p, dL/dv_p of state t (m_p / M_k); dL/dW = sum_t,r g_pre z^T, dL/db = sum g_pre.
// ------------------------------------------------------------------------------------
// segmented warp sum of NV values per distinct key (key < 0: no contribution), one global
// atomic per distinct key and value; all 32 lanes call it
template <int NV>
__device__ __forceinline__ void warp_key_add(int key, const float (&v)[NV], float* dst, int stride) {
  const int lane = threadIdx.x & 31;
  unsigned todo = __ballot_sync(0xffffffffu, key >= 0);
  while (todo) {
    const int src = __ffs(todo) - 1;
    const int k0 = __shfl_sync(0xffffffffu, key, src);
    const bool mine = key == k0;
    todo &= ~__ballot_sync(0xffffffffu, mine);
#pragma unroll
    for (int c = 0; c < NV; ++c) {
      float s = mine ? v[c] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == src) atomicAdd(&dst[(size_t)k0 * stride + c], s);
    }
  }
}

// z value j of rollout r from the group sums acc[B][K][2D] (m x, m v) and 1/M_k
template <int D>
__device__ __forceinline__ float ctrl_z(const KParams& P, int r, int j, const float* target, const float* acc,
                                        const float* Minv) {
  if (j < D) return target[j];
  j -= D;
  const int half = P.K * D;
  const int v = j >= half;
  if (v) j -= half;
  const int k = j / D, a = j % D;
  return __ldcg(&acc[((size_t)r * P.K + k) * 2 * D + v * D + a]) * Minv[r * P.K + k];
}

template <int D>
__global__ __launch_bounds__(256) void k_ctrl_observe(KParams P, const float* __restrict__ st,
                                                      const int* __restrict__ orig, const float4* __restrict__ prm,
                                                      const int* __restrict__ aid, float* acc, int* counter,
                                                      const float* __restrict__ W, const float* __restrict__ b,
                                                      const float* __restrict__ target, const float* __restrict__ Minv,
                                                      float* __restrict__ act, float* __restrict__ z_t, int t) {
  MPM_PDL_ENTRY();
  __shared__ int s_last;
  const size_t NT = P.NT;
  for (int j0 = blockIdx.x * blockDim.x; j0 < P.NT; j0 += gridDim.x * blockDim.x) {  // warp-uniform trips
    const int j = j0 + threadIdx.x;
    int key = -1;
    float val[2 * D];
#pragma unroll
    for (int c = 0; c < 2 * D; ++c) val[c] = 0.f;
    if (j < P.NT) {
      const int u = orig[j];
      const int k = aid[u];
      if (k >= 0) {
        key = (j / P.N) * P.K + k;
        const float m = prm[u].x;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          val[a] = m * st[rix<D>(comp_x<D>(a), j, NT)];
          val[D + a] = m * st[rix<D>(comp_v<D>(a), j, NT)];
        }
      }
    }
    warp_key_add<2 * D>(key, val, acc, 2 * D);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(counter, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int KD = P.K * D;
  for (int idx = threadIdx.x; idx < P.B * KD; idx += blockDim.x) {
    const int r = idx / KD, i = idx % KD;
    float pre = b[i];
    for (int jz = 0; jz < P.nz; ++jz) pre = fmaf(W[(size_t)i * P.nz + jz], ctrl_z<D>(P, r, jz, target, acc, Minv), pre);
    act[(((size_t)r * P.T + t) * P.K) * D + i] = tanhf(pre);
  }
  for (int idx = threadIdx.x; idx < P.B * P.nz; idx += blockDim.x)
    z_t[idx] = ctrl_z<D>(P, idx / P.nz, idx % P.nz, target, acc, Minv);
  __syncthreads();
  for (int idx = threadIdx.x; idx < P.B * P.K * 2 * D; idx += blockDim.x) acc[idx] = 0.f;
  if (threadIdx.x == 0) *counter = 0;
}

// one CTA per rollout: g_pre (taped) and dL/dz = W^T g_pre
template <int D>
__global__ __launch_bounds__(256) void k_ctrl_adj_param(KParams P, const float* __restrict__ da,
                                                        const float* __restrict__ act, const float* __restrict__ W,
                                                        float* __restrict__ gpre_t, float* __restrict__ gz, int t) {
  MPM_PDL_ENTRY();
  extern __shared__ float s_gpre[];  // [K D]
  const int r = blockIdx.x, KD = P.K * D;
  for (int i = threadIdx.x; i < KD; i += blockDim.x) {
    const size_t o = (((size_t)r * P.T + t) * P.K) * D + i;
    const float a = act[o];
    const float g = da[o] * (1.f - a * a);
    s_gpre[i] = g;
    gpre_t[(size_t)r * KD + i] = g;
  }
  __syncthreads();
  for (int jz = threadIdx.x; jz < P.nz; jz += blockDim.x) {
    float acc = 0.f;
    for (int i = 0; i < KD; ++i) acc = fmaf(W[(size_t)i * P.nz + jz], s_gpre[i], acc);
    gz[(size_t)r * P.nz + jz] = acc;
  }
}

// dL/dz -> dL/dx_p, dL/dv_p of state t (storage order t), closed-loop term
template <int D>
__global__ void k_ctrl_adj_state(KParams P, const float* __restrict__ gz, const int* __restrict__ orig,
                                 const float4* __restrict__ prm, const int* __restrict__ aid,
                                 const float* __restrict__ Minv, float* __restrict__ g) {
  MPM_PDL_ENTRY();
  const size_t NT = P.NT;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P.NT; j += gridDim.x * blockDim.x) {
    const int u = orig[j];
    const int k = aid[u];
    if (k < 0) continue;
    const int r = j / P.N;
    const float w = prm[u].x * Minv[r * P.K + k];
    const float* z = gz + (size_t)r * P.nz + D;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      g[rix<D>(comp_x<D>(a), j, NT)] += w * z[k * D + a];
      g[rix<D>(comp_v<D>(a), j, NT)] += w * z[P.K * D + k * D + a];
    }
  }
}

// end of the backward: dL/dW[i][jz] = sum_{t,r} g_pre[t][r][i] z[t][r][jz], dL/db, dL/dtarget
template <int D>
__global__ void k_ctrl_adj_reduce(KParams P, int T, const float* __restrict__ gpre, const float* __restrict__ z,
                                  const float* __restrict__ W, float* __restrict__ gW, float* __restrict__ gb,
                                  float* __restrict__ gtarget) {
  const int KD = P.K * D, n = KD * P.nz;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n + KD + D; idx += gridDim.x * blockDim.x) {
    float acc = 0.f;
    if (idx < n) {
      const int i = idx / P.nz, jz = idx % P.nz;
      for (int q = 0; q < T * P.B; ++q) acc = fmaf(gpre[(size_t)q * KD + i], z[(size_t)q * P.nz + jz], acc);
      gW[idx] = acc;
    } else if (idx < n + KD) {
      const int i = idx - n;
      for (int q = 0; q < T * P.B; ++q) acc += gpre[(size_t)q * KD + i];
      gb[i] = acc;
    } else {
      const int a = idx - n - KD;  // target enters z[0:D]: dL/dtarget = sum W[:, a]^T g_pre
      for (int q = 0; q < T * P.B; ++q)
        for (int i = 0; i < KD; ++i) acc = fmaf(W[(size_t)i * P.nz + a], gpre[(size_t)q * KD + i], acc);
      gtarget[a] = acc;
    }
  }
}

// group masses M[r][k] (and counts) for 1/M_k
__global__ void k_ctrl_mass(int NT, int N, int K, const float4* __restrict__ prm, const int* __restrict__ aid,
                            float* __restrict__ M, int* __restrict__ cnt) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < NT; u += gridDim.x * blockDim.x) {
    const int k = aid[u];
    if (k < 0) continue;
    atomicAdd(&M[(u / N) * K + k], prm[u].x);
    atomicAdd(&cnt[(u / N) * K + k], 1);
  }
}

// NEXT N2: at a segment boundary the recomputed forward may order state t differently from the
// run whose adjoint is carried in (a last-bit change of x from the order of P2G's float atomics
// can move a particle across a cell boundary): remap the adjoint through the user order.
__global__ void k_invert_perm(int NT, const int* __restrict__ orig, int* __restrict__ inv) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < NT; j += gridDim.x * blockDim.x) inv[orig[j]] = j;
}
__global__ void k_remap_adjoint(int NT, int S, const int* __restrict__ old_orig, const int* __restrict__ inv_new,
                                const float* __restrict__ src, float* __restrict__ dst) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < NT; j += gridDim.x * blockDim.x) {
    const int jn = inv_new[old_orig[j]];
    for (int c = 0; c < S; ++c) dst[rixs(S, c, jn, NT)] = src[rixs(S, c, j, NT)];
  }
}

// ------------------------------------------------------------------------------------
// Slab mode.  A rank owns the particles of one x-slab; the only nodes two ranks
// can both touch lie in a window of block-planes around each slab boundary, and the only
// exchange is the symmetric sum of those windows (after P2G in the forward, after G2P^T in
// the backward).  Block-linear order has axis 0 slowest, so a window of block-planes
// [bx0, bx0 + nwp) is the contiguous block range [bx0 nbpa^(D-1), (bx0 + nwp) nbpa^(D-1)).
// pack: window blocks -> dense buffer (0 where this rank has no slot); unpack: grid += buffer
// where this rank has a slot (a node it never reads needs no value).  Both ranks add the
// same two partial sums, so their copies of a window node are bitwise equal.
// grid index of slot s = (s - sub) * 64 + l, sub = 0 (tape arena) or the step base (adjoint).
// ------------------------------------------------------------------------------------
__global__ void k_band_pack(int nblk, int gb_lo, int gb_hi, const int* __restrict__ slot_of,
                            const int* __restrict__ info_t, int adj, const float4* __restrict__ g,
                            float4* __restrict__ out_lo, float4* __restrict__ out_hi) {
  MPM_PDL_ENTRY();
  const int sub = adj ? info_t[I_BASE] : 0;
  const int n = nblk * kCPB;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n; i += gridDim.x * blockDim.x) {
    const bool hi = i >= n;
    float4* out = hi ? out_hi : out_lo;
    if (!out) continue;
    const int e = hi ? i - n : i;
    const int s = __ldg(&slot_of[(hi ? gb_hi : gb_lo) + e / kCPB]);
    out[e] = s >= 0 ? g[(size_t)(s - sub) * kCPB + e % kCPB] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

__global__ void k_band_unpack(int nblk, int gb_lo, int gb_hi, const int* __restrict__ slot_of,
                              const int* __restrict__ info_t, int adj, float4* __restrict__ g,
                              const float4* __restrict__ in_lo, const float4* __restrict__ in_hi) {
  MPM_PDL_ENTRY();
  const int sub = adj ? info_t[I_BASE] : 0;
  const int n = nblk * kCPB;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n; i += gridDim.x * blockDim.x) {
    const bool hi = i >= n;
    const float4* in = hi ? in_hi : in_lo;
    if (!in) continue;
    const int e = hi ? i - n : i;
    const int s = __ldg(&slot_of[(hi ? gb_hi : gb_lo) + e / kCPB]);
    if (s < 0) continue;
    float4& q = g[(size_t)(s - sub) * kCPB + e % kCPB];
    const float4 r = in[e];
    q = make_float4(q.x + r.x, q.y + r.y, q.z + r.z, q.w + r.w);
  }
}

// ------------------------------------------------------------------------------------
// Migrating slab mode (SURVEY 8e "migrating particles"): a particle is owned, at every step, by
// the slab whose [own_lo, own_hi) holds its base_x.  After G2P of step t the particles that left
// (mig_pack, in g2p_particle) sit in the send buffers; the neighbours' buffers are received and
// appended behind the n_t particles G2P wrote (storage slots [n_t, n_t + a_L + a_R) of state
// t+1, left arrivals first).  The send buffers stay on the tape: the backward sends the adjoint
// of every arrival slot back to the rank it came from and writes the adjoints coming back into
// the slots the leavers left (their sorted slots k, recorded in the records).
// ------------------------------------------------------------------------------------
// after G2P of step t: the particles of state t+1 (slots [0, n_t)) whose base_x left the slab
// become holes (kDeadKey, taken out of the block histogram G2P built) and their records go to
// the send buffer of that side (record order = arrival order at the neighbour)
template <int D>
__global__ void k_mig_leavers(KParams P, MigParams M, const int* __restrict__ block_start_t, const float* __restrict__ st_next,
                              const int* __restrict__ orig_next, int* __restrict__ key, int* __restrict__ cnt,
                              float* __restrict__ send_l, float* __restrict__ send_r, ErrLatch* err, int t) {
  MPM_PDL_ENTRY();
  using MG = Mig<D>;
  const int nt = block_start_t[P.NBT];
  const size_t NT = P.NT;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nt; j += gridDim.x * blockDim.x) {
    const int bx = base_of(st_next[rix<D>(comp_x<D>(0), j, NT)], P.fres);
    if (bx >= M.own_lo && bx < M.own_hi) continue;
    const int kj = key[j];
    if (kj >= 0) atomicSub(&cnt[kj / kCPB], 1);
    key[j] = kDeadKey;
    float* buf = bx < M.own_lo ? send_l : send_r;
    const int pos = atomicAdd(reinterpret_cast<int*>(buf), 1);
    if (pos >= M.mig_cap) {
      latch(err, E_MIGRATE, t + 1, orig_next[j]);
      continue;
    }
    float* rec = buf + MG::HDR + (size_t)pos * MG::R;
    for (int c = 0; c < MG::S; ++c) rec[c] = st_next[rix<D>(c, j, NT)];
    rec[MG::U] = __int_as_float(orig_next[j]);
    rec[MG::K] = __int_as_float(j);
  }
}

template <int D>
__global__ void k_mig_append(KParams P, MigParams M, const float* __restrict__ recv_l, const float* __restrict__ recv_r,
                             const int* __restrict__ block_start_t, float* __restrict__ st_next,
                             int* __restrict__ orig_next, int* __restrict__ key, int* __restrict__ cnt,
                             int* __restrict__ info_next, ErrLatch* err, int t) {
  MPM_PDL_ENTRY();
  using MG = Mig<D>;
  const int nt = block_start_t[P.NBT];  // particles G2P wrote (live at step t)
  const int al = recv_l ? min(*reinterpret_cast<const int*>(recv_l), M.mig_cap) : 0;
  const int ar = recv_r ? min(*reinterpret_cast<const int*>(recv_r), M.mig_cap) : 0;
  const size_t NT = P.NT;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (nt + al + ar > P.NT) latch(err, E_MIGRATE, t + 1, nt + al + ar);
    info_next[I_NSLOT] = min(nt + al + ar, P.NT);
  }
  for (int i0 = blockIdx.x * blockDim.x; i0 < al + ar; i0 += gridDim.x * blockDim.x) {  // warp-uniform trips
    const int i = i0 + threadIdx.x;
    const int j = nt + i;
    bool valid = i < al + ar && j < P.NT;
    int gb = 0;
    if (valid) {
      const float* rec = (i < al ? recv_l + MG::HDR + (size_t)i * MG::R : recv_r + MG::HDR + (size_t)(i - al) * MG::R);
      for (int c = 0; c < MG::S; ++c) st_next[rix<D>(c, j, NT)] = rec[c];
      orig_next[j] = __float_as_int(rec[MG::U]);
      float x[D];
#pragma unroll
      for (int a = 0; a < D; ++a) x[a] = rec[comp_x<D>(a)];
      int k;
      if (const int e = key_of<D>(x, 0, P, gb, k)) latch(err, e, t + 1, orig_next[j]);
      const int bx = base_of(x[0], P.fres);
      if (bx < M.own_lo || bx >= M.own_hi) latch(err, E_MIGRATE, t + 1, orig_next[j]);  // crossed a whole slab
      key[j] = k;
    }
    warp_hist_add(cnt, gb, valid);
  }
}

// backward, before G2P^T of step t: the adjoint of state t+1 at this rank's arrival slots goes
// back to the sender (left arrivals to the left, right ones to the right, in arrival order)
template <int D>
__global__ void k_mig_rev_pack(KParams P, MigParams M, const float* __restrict__ recv_l, const float* __restrict__ recv_r,
                               const int* __restrict__ block_start_t, const float* __restrict__ g,
                               float* __restrict__ out_l, float* __restrict__ out_r) {
  MPM_PDL_ENTRY();
  using MG = Mig<D>;
  const int nt = block_start_t[P.NBT];
  const int al = recv_l ? min(*reinterpret_cast<const int*>(recv_l), M.mig_cap) : 0;
  const int ar = recv_r ? min(*reinterpret_cast<const int*>(recv_r), M.mig_cap) : 0;
  const size_t NT = P.NT;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < (al + ar) * MG::S; q += gridDim.x * blockDim.x) {
    const int i = q / MG::S, c = q - i * MG::S;
    const int j = nt + i;
    if (j >= P.NT) continue;
    float* out = i < al ? out_l + (size_t)i * MG::S : out_r + (size_t)(i - al) * MG::S;
    out[c] = g[rix<D>(c, j, NT)];
  }
}

// ... and the adjoints coming back from the neighbours fill the slots of this rank's leavers
template <int D>
__global__ void k_mig_rev_unpack(KParams P, MigParams M, const float* __restrict__ sent_l, const float* __restrict__ sent_r,
                                 const float* __restrict__ in_l, const float* __restrict__ in_r, float* __restrict__ g) {
  MPM_PDL_ENTRY();
  using MG = Mig<D>;
  const int nl = sent_l ? min(*reinterpret_cast<const int*>(sent_l), M.mig_cap) : 0;
  const int nr = sent_r ? min(*reinterpret_cast<const int*>(sent_r), M.mig_cap) : 0;
  const size_t NT = P.NT;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < (nl + nr) * MG::S; q += gridDim.x * blockDim.x) {
    const int i = q / MG::S, c = q - i * MG::S;
    const float* rec = i < nl ? sent_l + MG::HDR + (size_t)i * MG::R : sent_r + MG::HDR + (size_t)(i - nl) * MG::R;
    const float* in = i < nl ? in_l + (size_t)i * MG::S : in_r + (size_t)(i - nl) * MG::S;
    const int k = __float_as_int(rec[MG::K]);
    g[rix<D>(c, k, NT)] = in[c];
  }
}

__global__ void k_add_inplace(size_t n, float* __restrict__ a, const float* __restrict__ b) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    a[i] += b[i];
}

// ------------------------------------------------------------------------------------
// grid^T: steps L (reverse wall order R6), D, E (R9).
// adjoint node (dL/dv_i) -> (dL/dp_i, dL/dm_i) in place, from the memo's (p, m).  Also
// prepares the other adjoint buffer for backward step t-1 (zero + reset its counters).
// ------------------------------------------------------------------------------------
template <int D>
__global__ void k_grid_adj(KParams P, const int* __restrict__ info_t, const int* __restrict__ touched_list,
                           const float4* __restrict__ arena, float4* __restrict__ ag,
                           int* __restrict__ info_prev, float4* __restrict__ ag_prev) {
  MPM_PDL_ENTRY();
  if (info_prev) adj_prepare(info_prev, ag_prev, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
  const int n = info_t[I_NTOUCH] * kCPB;
  const float4* g = arena + (size_t)info_t[I_BASE] * kCPB;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float4 q = g[i];  // (p, m)
    const float4 a = ag[i];
    float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
    if (q.w > 0.f) {
      const int gb = touched_list[i / kCPB];
      const int r = gb / P.nb;
      int node[D];
      {
        int t = gb - r * P.nb, l = i % kCPB;
#pragma unroll
        for (int d = D - 1; d >= 0; --d) {
          node[d] = (t % P.nbpa) * Dim<D>::BB + l % Dim<D>::BB;
          t /= P.nbpa;
          l /= Dim<D>::BB;
        }
      }
      const float im = 1.f / q.w;
      float vb[D] = {}, gv[D] = {};
      vb[0] = fmaf(q.x, im, P.dt * P.g[0]); vb[1] = fmaf(q.y, im, P.dt * P.g[1]);
      gv[0] = a.x; gv[1] = a.y;
      if (D == 3) { vb[D - 1] = fmaf(q.z, im, P.dt * P.g[2]); gv[D - 1] = a.z; }
      if (in_band<D>(node, P.res, P.bound)) project_node_adj<D>(vb, gv, node, P);
      // gravity adjoint = identity (R5); vbar = p/m + dt g -> dp = gv/m, dm = -(p . gv)/m^2
      float pg = 0.f;
#pragma unroll
      for (int d = 0; d < D; ++d) pg = fmaf(vb[d] - P.dt * P.g[d], gv[d], pg);
      out.x = gv[0] * im;
      out.y = gv[1] * im;
      if (D == 3) out.z = gv[D - 1] * im;
      out.w = -pg * im;
    }
    ag[i] = out;
  }
}

// ------------------------------------------------------------------------------------
// seed, readback, finalize
// ------------------------------------------------------------------------------------
// user-order AoS seed -> SoA adjoint in storage order t (orig_t maps storage -> user);
// accumulate = add to the adjoint already there (per-step seeds of a running loss, N4)
template <int D>
__global__ void k_seed(KParams P, const int* __restrict__ orig, const float* __restrict__ gx,
                       const float* __restrict__ gv, const float* __restrict__ gF,
                       const float* __restrict__ gC, float* __restrict__ g, int accumulate,
                       const int* __restrict__ nslot) {
  MPM_PDL_ENTRY();
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (nslot ? *nslot : P.NT)) return;  // migrating slab mode: the state's storage slots
  const size_t NT = P.NT;
  int u = orig[k];
  auto put = [&](int comp, float val) {
    float* q = &g[rix<D>(comp, k, NT)];
    *q = accumulate ? *q + val : val;
  };
#pragma unroll
  for (int a = 0; a < D; ++a) {
    put(comp_x<D>(a), gx ? gx[u * D + a] : 0.f);
    put(comp_v<D>(a), gv ? gv[u * D + a] : 0.f);
#pragma unroll
    for (int b = 0; b < D; ++b) {
      put(comp_F<D>(a, b), gF ? gF[(u * D + a) * D + b] : 0.f);
      put(comp_C<D>(a, b), gC ? gC[(u * D + a) * D + b] : 0.f);
    }
  }
}

// SoA storage order -> user AoS (x, v, F, C), any may be null.  Migrating slab mode: only the
// slots [0, *nslot) whose particle this slab owns in `owner` (the state's positions) are written.
template <int D>
__global__ void k_soa_to_user(KParams P, const int* __restrict__ orig, const float* __restrict__ st,
                              float* x, float* v, float* F, float* C, int state,
                              const int* __restrict__ nslot = nullptr, const float* __restrict__ owner = nullptr,
                              MigParams M = MigParams{}) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= (nslot ? *nslot : P.NT)) return;
  const size_t NT = P.NT;
  if (owner) {
    const int bx = base_of(owner[rix<D>(comp_x<D>(0), j, NT)], P.fres);
    if (bx < M.own_lo || bx >= M.own_hi) return;  // a hole: the particle is the neighbour's now
  }
  int u = orig ? orig[j] : j;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (x) x[u * D + a] = st[rix<D>(comp_x<D>(a), j, NT)];
    if (v) v[u * D + a] = st[rix<D>(comp_v<D>(a), j, NT)];
#pragma unroll
    for (int b = 0; b < D; ++b) {
      // states store H = F - I; adjoints (dL/dF = dL/dH) are returned as they are
      if (F) F[(u * D + a) * D + b] = st[rix<D>(comp_F<D>(a, b), j, NT)] + ((state && a == b) ? 1.f : 0.f);
      if (C) C[(u * D + a) * D + b] = st[rix<D>(comp_C<D>(a, b), j, NT)];
    }
  }
}

__global__ void k_finalize_params(int NT, const float* __restrict__ E, const float* __restrict__ nu,
                                  const float* __restrict__ dmu, const float* __restrict__ dlam,
                                  float* dE, float* dnu) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= NT) return;
  // R19: chain through the Lame parameters
  float e = E[j], n = nu[j], gm = dmu[j], gl = dlam[j];
  float a = 1.f + n, b = 1.f - 2.f * n;
  if (dE) dE[j] = gm / (2.f * a) + gl * n / (a * b);
  if (dnu) dnu[j] = -gm * e / (2.f * a * a) + gl * e * (1.f + 2.f * n * n) / (a * a * b * b);
}

// dense readback of the tape grid of one step: [B][res^D] (m, vbar)
template <int D>
__global__ void k_dense_grid(KParams P, const int* __restrict__ info_t, const int* __restrict__ touched_list,
                             const float4* __restrict__ arena, float* m, float* vbar) {
  const int n = info_t[I_NTOUCH] * kCPB;
  const float4* g = arena + (size_t)info_t[I_BASE] * kCPB;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int gb = touched_list[i / kCPB];
    const int r = gb / P.nb;
    int t = gb - r * P.nb, l = i % kCPB;
    int node[D];
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      node[d] = (t % P.nbpa) * Dim<D>::BB + l % Dim<D>::BB;
      t /= P.nbpa;
      l /= Dim<D>::BB;
    }
    size_t lin = 0;
#pragma unroll
    for (int d = 0; d < D; ++d) lin = lin * P.res + node[d];
    size_t nn = 1;
#pragma unroll
    for (int d = 0; d < D; ++d) nn *= P.res;
    size_t o = (size_t)r * nn + lin;
    float4 q = g[i];  // (p, m)
    if (m) m[o] = q.w;
    if (vbar && q.w > 0.f) {
      vbar[o * D + 0] = q.x / q.w + P.dt * P.g[0];
      vbar[o * D + 1] = q.y / q.w + P.dt * P.g[1];
      if (D == 3) vbar[o * D + D - 1] = q.z / q.w + P.dt * P.g[2];
    }
  }
}

}  // namespace mpm
