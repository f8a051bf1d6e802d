/*
 * mpm_oracle.h -- plain, slow, obviously-correct CPU oracle for the differentiable
 * MLS-MPM step of ChainQueen (arXiv 1810.01054).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  The product
 * path (paper_1810_01054_b200/) never links, imports or executes anything here; it
 * shares no code, header, table or constant generator with this file.
 *
 * Precision: fp64 throughout, except binning, which decides integers from the fp32
 * positions the CUDA path stores (reading R17: the decision is taken in the
 * kernel's precision; for power-of-two res it is exact in both).
 *
 * Citations: "P:<line>" is /root/reference/PAPER.md line <line>; "R<k>" is reading k of
 * DESIGN.md section "Readings of the paper".
 *
 * State record of one particle (S = 2d + 2d^2 doubles):  x[d], v[d], C[d][d], F[d][d],
 * matrices row-major (C[a][b] at C[a*d+b]).
 */
#ifndef MPM_ORACLE_H
#define MPM_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int dim;             /* 2 or 3                                                    */
  int res;             /* nodes per axis; dx = 1/res; domain [0,1)^d                */
  int n;               /* particles (one rollout)                                   */
  int n_act;           /* K actuators; actuation array is [T][K][dim]               */
  double dt;
  double gravity[3];
  int bound;           /* wall band width in nodes (R6)                             */
  double friction[6];  /* c per wall (-x,+x,-y,+y,-z,+z); c < 0 => sticky (R6)     */
  double act_strength; /* s in sigma_pa = s * Diag(a)  (R4)                         */
  double eps;          /* epsilon of step L (R7)                                    */
  int material;        /* 0 = neo-Hookean (R1), 1 = fixed-corotated (NEXT N3, R21)   */
} orc_cfg;

enum { ORC_OK = 0, ORC_ERR_OUT_OF_DOMAIN = 1, ORC_ERR_INVERTED = 2, ORC_ERR_ARG = 3 };

/* ---- unit pieces (exported so the pins in tests/ can reach them) ---- */
double orc_N(double u);        /* quadratic B-spline N(u), R2 */
double orc_dN(double u);       /* dN/du                        */
int    orc_weights(double xg, int* base, double w[3], double dw[3]);
double orc_det(int dim, const double* F);
void   orc_inv(int dim, const double* F, double* Finv);
double orc_psi(int dim, const double* F, double mu, double lam);           /* R1 */
void   orc_pk1(int dim, const double* F, double mu, double lam, double* P); /* R1 */
void   orc_dPdF(int dim, const double* F, double mu, double lam, double* H);/* H[g][e][a][b] = dP_ge/dF_ab */
/* fixed-corotated (NEXT N3, R21): psi = mu |F - R|^2 + lam/2 (J - 1)^2,
 * P = 2 mu (F - R) + lam (J - 1) J F^-T, R the rotation of the polar decomposition F = R S */
int    orc_polar(int dim, const double* F, double* R);
double orc_psi_fcr(int dim, const double* F, double mu, double lam);
void   orc_pk1_fcr(int dim, const double* F, double mu, double lam, double* P);
void   orc_dPdF_fcr(int dim, const double* F, double mu, double lam, double* H);
void   orc_lame(double E, double nu, double* mu, double* lam);
void   orc_project(int dim, const double* v, const double* nrm, double c, double eps, double* vstar);
void   orc_project_adj(int dim, const double* v, const double* nrm, double c, double eps,
                       const double* dvstar, double* dv);
void   orc_grid_node(const orc_cfg* cfg, const int* node, double m, const double* p,
                     double* vbar, double* v);
void   orc_grid_node_adj(const orc_cfg* cfg, const int* node, double m, const double* p,
                         const double* dv, double* dp, double* dm);

/* Grid of one step (P2G Eqs. 3-5, then Eq. 6 + R5/R6): m [res^d], p / vbar / v [res^d][dim].
 * Node linear index = row-major over (i_0, ..., i_{d-1}).                              */
int orc_step_grid(const orc_cfg* cfg, const double* state, const double* mass,
                  const double* vol, const double* E, const double* nu, const int* act_id,
                  const double* act_t, double* m, double* p, double* vbar, double* v);

/* ---- one rollout, whole trajectory ---- */
/* traj: [(n_steps+1)][n][S]; traj[0] is the input state; fills traj[1..n_steps].
 * act: [n_steps][K][dim] (may be NULL when K == 0).  act_id[p] in [-1, K).
 * err_index (may be NULL) receives (step, particle) of the first error.              */
int orc_forward(const orc_cfg* cfg, int n_steps, double* traj,
                const double* mass, const double* vol, const double* E, const double* nu,
                const int* act_id, const double* act, int* err_index);

/* Reverse-mode over the whole trajectory, P:165 ("applying the chain rule at a higher
 * level from the final state all-the-way to the initial state").
 * seed: dL/dstate_T [n][S].  grad0: dL/dstate_0 [n][S].  gE, gnu: [n] (overwritten).
 * ga: [n_steps][K][dim] (overwritten; may be NULL when K == 0).                      */
int orc_backward(const orc_cfg* cfg, int n_steps, const double* traj,
                 const double* mass, const double* vol, const double* E, const double* nu,
                 const int* act_id, const double* act, const double* seed,
                 double* grad0, double* gE, double* gnu, double* ga);

/* As orc_backward, with a seed for EVERY state (seeds [(n_steps+1)][n][S]: a running loss
 * sum_t L_t(state_t), NEXT N4) and the mass gradient gm [n] (NEXT N3; NULL = skip).      */
int orc_backward_ex(const orc_cfg* cfg, int n_steps, const double* traj,
                    const double* mass, const double* vol, const double* E, const double* nu,
                    const int* act_id, const double* act, const double* seeds,
                    double* grad0, double* gE, double* gnu, double* ga, double* gm);

/* Binning (north_star item 1), decided on fp32 positions.
 * x: [batch][n][dim] fp32.  key: [batch*n].  perm: [batch*n] (sorted slot -> index).
 * block_start: [batch*nb + 1], nb = (res/Bb)^dim, Bb = 4 (3D) / 8 (2D).              */
int orc_bin(int dim, int res, int batch, int n, const float* x,
            int* key, int* perm, int* block_start);

#ifdef __cplusplus
}
#endif
#endif
