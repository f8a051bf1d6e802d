/*
 * mpm_oracle.c -- plain, slow, obviously-correct CPU oracle (fp64) for the differentiable
 * MLS-MPM step of ChainQueen (arXiv 1810.01054).
 *
 * TEST INFRASTRUCTURE ONLY (see mpm_oracle.h).  The CUDA product path shares no code with
 * this file.  Every loop below is written in the order and notation of the paper:
 *   forward   P:131-153 (Eqs. 3-10) and the supplement's restatement P:429-437 (S1-S8);
 *   backward  supplement steps A-L, in the order of P:490-491;
 *   chain over steps.
 * Where the paper is silent or garbled the DESIGN.md reading R<k> is cited.
 *
 * Pinning (see tests/test_oracle_*.py): every function here is checked against something
 * other than itself -- printed values (tests/golden/), closed forms, conservation laws,
 * central finite differences in fp64 and the exact closed-form CoM gradient.
 */
#include "mpm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define MAXD 3

/* ------------------------------------------------------------------------------------ */
/* Kernel N: the quadratic B-spline (P:113 names it; formula not printed -> R2).        */
/* N(u) = 3/4 - u^2 for |u| < 1/2;  (3/2 - |u|)^2 / 2 for 1/2 <= |u| < 3/2;  0 otherwise */
/* ------------------------------------------------------------------------------------ */
double orc_N(double u) {
  double a = fabs(u);
  if (a < 0.5) return 0.75 - a * a;
  if (a < 1.5) return 0.5 * (1.5 - a) * (1.5 - a);
  return 0.0;
}

double orc_dN(double u) {
  double a = fabs(u);
  double s = (u < 0.0) ? -1.0 : 1.0;
  if (a < 0.5) return -2.0 * u;
  if (a < 1.5) return -(1.5 - a) * s;
  return 0.0;
}

/* Stencil of one axis.  xg = x/dx.  base = floor(xg - 1/2) (R2); the three nodes
 * base+o, o = 0,1,2, get w[o] = N(xg - (base+o)) and dw[o] = N'(xg - (base+o)).
 * Returns 0; base is written unconditionally (range checked by the caller).           */
int orc_weights(double xg, int* base, double w[3], double dw[3]) {
  int b = (int)floor(xg - 0.5);
  for (int o = 0; o < 3; ++o) {
    double u = xg - (double)(b + o);
    w[o] = orc_N(u);
    dw[o] = orc_dN(u);
  }
  *base = b;
  return 0;
}

/* ------------------------------------------------------------------------------------ */
/* small dense linear algebra, written out                                              */
/* ------------------------------------------------------------------------------------ */
double orc_det(int dim, const double* F) {
  if (dim == 2) return F[0] * F[3] - F[1] * F[2];
  return F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
         F[2] * (F[3] * F[7] - F[4] * F[6]);
}

void orc_inv(int dim, const double* F, double* Fi) {
  double J = orc_det(dim, F);
  if (dim == 2) {
    Fi[0] = F[3] / J;
    Fi[1] = -F[1] / J;
    Fi[2] = -F[2] / J;
    Fi[3] = F[0] / J;
    return;
  }
  /* adjugate / det */
  Fi[0] = (F[4] * F[8] - F[5] * F[7]) / J;
  Fi[1] = (F[2] * F[7] - F[1] * F[8]) / J;
  Fi[2] = (F[1] * F[5] - F[2] * F[4]) / J;
  Fi[3] = (F[5] * F[6] - F[3] * F[8]) / J;
  Fi[4] = (F[0] * F[8] - F[2] * F[6]) / J;
  Fi[5] = (F[2] * F[3] - F[0] * F[5]) / J;
  Fi[6] = (F[3] * F[7] - F[4] * F[6]) / J;
  Fi[7] = (F[1] * F[6] - F[0] * F[7]) / J;
  Fi[8] = (F[0] * F[4] - F[1] * F[3]) / J;
}

/* Lame parameters from (E, nu), R1 (same formulas in 2D: plane strain). */
void orc_lame(double E, double nu, double* mu, double* lam) {
  *mu = E / (2.0 * (1.0 + nu));
  *lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
}

/* ------------------------------------------------------------------------------------ */
/* Constitutive model ("PK1 stress (dpsi/dF)"; psi not named -> R1 neo-Hookean) */
/*   psi = mu/2 (tr(F^T F) - d) - mu ln J + lam/2 (ln J)^2                                */
/*   P   = dpsi/dF = mu (F - F^-T) + lam ln J F^-T                                        */
/* ------------------------------------------------------------------------------------ */
double orc_psi(int dim, const double* F, double mu, double lam) {
  double tr = 0.0;
  for (int i = 0; i < dim * dim; ++i) tr += F[i] * F[i];
  double lnJ = log(orc_det(dim, F));
  return 0.5 * mu * (tr - (double)dim) - mu * lnJ + 0.5 * lam * lnJ * lnJ;
}

void orc_pk1(int dim, const double* F, double mu, double lam, double* P) {
  double Fi[9];
  orc_inv(dim, F, Fi);
  double lnJ = log(orc_det(dim, F));
  for (int a = 0; a < dim; ++a)
    for (int b = 0; b < dim; ++b) {
      double FinvT_ab = Fi[b * dim + a];
      P[a * dim + b] = mu * (F[a * dim + b] - FinvT_ab) + lam * lnJ * FinvT_ab;
    }
}

/* H[g][e][a][b] = d P_ge / d F_ab = d^2 psi / dF_ge dF_ab  (the Hessian of step H).
 * With Fi = F^-1:  mu d_ga d_eb + (mu - lam lnJ) Fi_ea Fi_bg + lam Fi_ba Fi_eg.            */
void orc_dPdF(int dim, const double* F, double mu, double lam, double* H) {
  double Fi[9];
  orc_inv(dim, F, Fi);
  double lnJ = log(orc_det(dim, F));
  int d = dim;
  for (int g = 0; g < d; ++g)
    for (int e = 0; e < d; ++e)
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
          double v = 0.0;
          if (g == a && e == b) v += mu;
          v += (mu - lam * lnJ) * Fi[e * d + a] * Fi[b * d + g];
          v += lam * Fi[b * d + a] * Fi[e * d + g];
          H[((g * d + e) * d + a) * d + b] = v;
        }
}

/* ------------------------------------------------------------------------------------ */
/* Fixed-corotated model (NEXT N3, DESIGN R21): the paper names no psi  */
/* (P:102-103); this is the second material the GPU offers.                               */
/*   F = R S (polar), psi = mu |F - R|^2 + lam/2 (J - 1)^2, P = 2 mu (F - R) + lam (J-1) J F^-T */
/* ------------------------------------------------------------------------------------ */

/* symmetric 3x3 eigen-decomposition by cyclic Jacobi rotations: A = Q diag(ev) Q^T */
static void jacobi3(const double* A_in, double* ev, double* Q) {
  double A[9];
  for (int i = 0; i < 9; ++i) { A[i] = A_in[i]; Q[i] = (i % 4 == 0) ? 1.0 : 0.0; }
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = A[1] * A[1] + A[2] * A[2] + A[5] * A[5];
    double nrm = A[0] * A[0] + A[4] * A[4] + A[8] * A[8];
    if (off <= 1e-34 * nrm) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double apq = A[p * 3 + q];
        if (apq == 0.0) continue;
        double theta = (A[q * 3 + q] - A[p * 3 + p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
        /* A <- J^T A J with J the rotation in the (p, q) plane */
        for (int k = 0; k < 3; ++k) {
          double akp = A[k * 3 + p], akq = A[k * 3 + q];
          A[k * 3 + p] = c * akp - sn * akq;
          A[k * 3 + q] = sn * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          double apk = A[p * 3 + k], aqk = A[q * 3 + k];
          A[p * 3 + k] = c * apk - sn * aqk;
          A[q * 3 + k] = sn * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          double qkp = Q[k * 3 + p], qkq = Q[k * 3 + q];
          Q[k * 3 + p] = c * qkp - sn * qkq;
          Q[k * 3 + q] = sn * qkp + c * qkq;
        }
      }
  }
  for (int i = 0; i < 3; ++i) ev[i] = A[i * 4];
}

/* R of F = R S with S symmetric positive definite (det F > 0).  2D: SPEC's closed form,
 * theta = atan2(F10 - F01, F00 + F11).  3D: S = (F^T F)^(1/2) by Jacobi, R = F S^-1. */
int orc_polar(int dim, const double* F, double* R) {
  if (!(orc_det(dim, F) > 0.0)) return ORC_ERR_INVERTED;
  if (dim == 2) {
    double th = atan2(F[2] - F[1], F[0] + F[3]);
    R[0] = cos(th); R[1] = -sin(th); R[2] = sin(th); R[3] = cos(th);
    return ORC_OK;
  }
  double FtF[9], ev[3], Q[9], Si[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int c = 0; c < 3; ++c) acc += F[c * 3 + a] * F[c * 3 + b];
      FtF[a * 3 + b] = acc;
    }
  jacobi3(FtF, ev, Q);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += Q[a * 3 + k] * Q[b * 3 + k] / sqrt(ev[k]);
      Si[a * 3 + b] = acc;
    }
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int c = 0; c < 3; ++c) acc += F[a * 3 + c] * Si[c * 3 + b];
      R[a * 3 + b] = acc;
    }
  return ORC_OK;
}

double orc_psi_fcr(int dim, const double* F, double mu, double lam) {
  double R[9];
  orc_polar(dim, F, R);
  double s = 0.0;
  for (int i = 0; i < dim * dim; ++i) s += (F[i] - R[i]) * (F[i] - R[i]);
  double J = orc_det(dim, F);
  return mu * s + 0.5 * lam * (J - 1.0) * (J - 1.0);
}

void orc_pk1_fcr(int dim, const double* F, double mu, double lam, double* P) {
  double R[9], Fi[9];
  orc_polar(dim, F, R);
  orc_inv(dim, F, Fi);
  double J = orc_det(dim, F);
  for (int a = 0; a < dim; ++a)
    for (int b = 0; b < dim; ++b)
      P[a * dim + b] = 2.0 * mu * (F[a * dim + b] - R[a * dim + b]) + lam * (J - 1.0) * J * Fi[b * dim + a];
}

/* dR for a perturbation dF (P:567's Hessian needs dR/dF):  with S = R^T F and
 * M = R^T dF,  R^T dR = [w]x  where  (tr(S) I - S) w = axial(M - M^T)  (3D; [w]x S + S [w]x
 * = [(tr(S) I - S) w]x for symmetric S), and w = (M_10 - M_01) / tr(S) in 2D. */
static void polar_dR(int d, const double* F, const double* R, const double* dF, double* dR) {
  double S[9], M[9], K[9];
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      double s = 0.0, m = 0.0;
      for (int c = 0; c < d; ++c) {
        s += R[c * d + a] * F[c * d + b];
        m += R[c * d + a] * dF[c * d + b];
      }
      S[a * d + b] = s;
      M[a * d + b] = m;
    }
  for (int i = 0; i < 9; ++i) K[i] = 0.0;
  if (d == 2) {
    double w = (M[2] - M[1]) / (S[0] + S[3]);
    K[1] = -w; K[3] = w;  /* [[0, -w], [w, 0]] in the 3x3 layout of K */
  } else {
    double ax[3] = {M[7] - M[5], M[2] - M[6], M[3] - M[1]}; /* axial(M - M^T) */
    double trS = S[0] + S[4] + S[8], A[9], Ai[9], w[3];
    for (int i = 0; i < 9; ++i) A[i] = -S[i];
    A[0] += trS; A[4] += trS; A[8] += trS;
    orc_inv(3, A, Ai);
    for (int a = 0; a < 3; ++a) w[a] = Ai[a * 3] * ax[0] + Ai[a * 3 + 1] * ax[1] + Ai[a * 3 + 2] * ax[2];
    K[1] = -w[2]; K[2] = w[1]; K[3] = w[2]; K[5] = -w[0]; K[6] = -w[1]; K[7] = w[0];
  }
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      double acc = 0.0;
      for (int c = 0; c < d; ++c) acc += R[a * d + c] * K[c * 3 + b];
      dR[a * d + b] = acc;
    }
}

/* H[g][e][a][b] = dP_ge/dF_ab = 2 mu (d_ga d_eb - dR_ge/dF_ab)
 *                + lam [ (J F^-T)_ge (J F^-T)_ab + (J - 1) J (Fi_ba Fi_eg - Fi_ea Fi_bg) ] */
void orc_dPdF_fcr(int dim, const double* F, double mu, double lam, double* H) {
  int d = dim;
  double R[9], Fi[9];
  orc_polar(d, F, R);
  orc_inv(d, F, Fi);
  double J = orc_det(d, F);
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      double dF[9] = {0}, dR[9];
      dF[a * d + b] = 1.0;
      polar_dR(d, F, R, dF, dR);
      for (int g = 0; g < d; ++g)
        for (int e = 0; e < d; ++e) {
          double v = 2.0 * mu * (((g == a && e == b) ? 1.0 : 0.0) - dR[g * d + e]);
          v += lam * (J * Fi[e * d + g]) * (J * Fi[b * d + a]);
          v += lam * (J - 1.0) * J * (Fi[b * d + a] * Fi[e * d + g] - Fi[e * d + a] * Fi[b * d + g]);
          H[((g * d + e) * d + a) * d + b] = v;
        }
    }
}

/* ------------------------------------------------------------------------------------ */
/* Friction projection, step L, forward definitions P:614-619 (R6, R7, R8).               */
/* ------------------------------------------------------------------------------------ */
void orc_project(int dim, const double* v, const double* n, double c, double eps, double* vs) {
  if (c < 0.0) { /* sticky wall (R6) */
    for (int a = 0; a < dim; ++a) vs[a] = 0.0;
    return;
  }
  double ln = 0.0; /* l_n = sum_a v_a n_a */
  for (int a = 0; a < dim; ++a) ln += v[a] * n[a];
  if (ln >= 0.0) { /* R8: identity branch (equal to the formula in real arithmetic) */
    for (int a = 0; a < dim; ++a) vs[a] = v[a];
    return;
  }
  double vt[MAXD], s = 0.0;
  for (int a = 0; a < dim; ++a) { vt[a] = v[a] - ln * n[a]; s += vt[a] * vt[a]; }
  double lt = sqrt(s + eps);
  double R = lt + c * fmin(ln, 0.0);
  double lts = fmax(R, 0.0);
  for (int a = 0; a < dim; ++a)
    vs[a] = lts * (vt[a] / lt) + fmax(ln, 0.0) * n[a];
}

/* Adjoint of orc_project, literally P:622-634, with H(x) = [x >= 0].          */
void orc_project_adj(int dim, const double* v, const double* n, double c, double eps,
                     const double* dvs, double* dv) {
  if (c < 0.0) {
    for (int a = 0; a < dim; ++a) dv[a] = 0.0;
    return;
  }
  double ln = 0.0;
  for (int a = 0; a < dim; ++a) ln += v[a] * n[a];
  if (ln >= 0.0) { /* R8 */
    for (int a = 0; a < dim; ++a) dv[a] = dvs[a];
    return;
  }
  double vt[MAXD], s = 0.0;
  for (int a = 0; a < dim; ++a) { vt[a] = v[a] - ln * n[a]; s += vt[a] * vt[a]; }
  double lt = sqrt(s + eps);
  double vhat[MAXD];
  for (int a = 0; a < dim; ++a) vhat[a] = vt[a] / lt;
  double R = lt + c * fmin(ln, 0.0);
  double lts = fmax(R, 0.0);
  double HR = (R >= 0.0) ? 1.0 : 0.0, Hmln = (-ln >= 0.0) ? 1.0 : 0.0, Hln = (ln >= 0.0) ? 1.0 : 0.0;

  double dlts = 0.0;
  for (int a = 0; a < dim; ++a) dlts += dvs[a] * vhat[a];
  double dvhat[MAXD];
  for (int a = 0; a < dim; ++a) dvhat[a] = dvs[a] * lts;
  double dlt = 0.0;
  for (int a = 0; a < dim; ++a) dlt += vt[a] * dvhat[a];
  dlt = -dlt / (lt * lt) + dlts * HR;
  double dvt[MAXD];
  for (int a = 0; a < dim; ++a) dvt[a] = (dlt * vt[a] + dvhat[a]) / lt;
  double dln = 0.0;
  for (int a = 0; a < dim; ++a) dln -= dvt[a] * n[a];
  dln += dlts * HR * c * Hmln;
  for (int a = 0; a < dim; ++a) dln += Hln * n[a] * dvs[a];
  for (int a = 0; a < dim; ++a) dv[a] = dln * n[a] + dvt[a];
}

/* ------------------------------------------------------------------------------------ */
/* Grid operation of one node: Eq. 6, then gravity (R5), then the wall-band  */
/* projections applied per axis in axis order (R6).  Nodes with m = 0 get 0 (R13).        */
/* ------------------------------------------------------------------------------------ */
static void wall_of(const orc_cfg* cfg, const int* node, int axis, int side, int* active,
                    double* n, double* c) {
  for (int a = 0; a < cfg->dim; ++a) n[a] = 0.0;
  *active = 0;
  if (side == 0 && node[axis] < cfg->bound) {
    *active = 1;
    n[axis] = 1.0;
    *c = cfg->friction[2 * axis];
  }
  if (side == 1 && node[axis] >= cfg->res - cfg->bound) {
    *active = 1;
    n[axis] = -1.0;
    *c = cfg->friction[2 * axis + 1];
  }
}

void orc_grid_node(const orc_cfg* cfg, const int* node, double m, const double* p,
                   double* vbar, double* v) {
  int d = cfg->dim;
  if (!(m > 0.0)) {
    for (int a = 0; a < d; ++a) vbar[a] = v[a] = 0.0;
    return;
  }
  for (int a = 0; a < d; ++a) vbar[a] = p[a] / m + cfg->dt * cfg->gravity[a];
  double cur[MAXD], nxt[MAXD];
  for (int a = 0; a < d; ++a) cur[a] = vbar[a];
  for (int axis = 0; axis < d; ++axis)
    for (int side = 0; side < 2; ++side) {
      int act;
      double n[MAXD], c = 0.0;
      wall_of(cfg, node, axis, side, &act, n, &c);
      if (!act) continue;
      orc_project(d, cur, n, c, cfg->eps, nxt);
      for (int a = 0; a < d; ++a) cur[a] = nxt[a];
    }
  for (int a = 0; a < d; ++a) v[a] = cur[a];
}

/* Adjoint of orc_grid_node: step L in reverse axis order (R6), gravity is a pass-through
 * (R5), then step D and step E's first form (R9).                    */
void orc_grid_node_adj(const orc_cfg* cfg, const int* node, double m, const double* p,
                       const double* dv_in, double* dp, double* dm) {
  int d = cfg->dim;
  if (!(m > 0.0)) {
    for (int a = 0; a < d; ++a) dp[a] = 0.0;
    *dm = 0.0;
    return;
  }
  /* replay the forward, remembering the input of every active projection */
  double stage_in[2 * MAXD][MAXD], stage_n[2 * MAXD][MAXD], stage_c[2 * MAXD];
  int ns = 0;
  double cur[MAXD], nxt[MAXD];
  for (int a = 0; a < d; ++a) cur[a] = p[a] / m + cfg->dt * cfg->gravity[a];
  for (int axis = 0; axis < d; ++axis)
    for (int side = 0; side < 2; ++side) {
      int act;
      double n[MAXD], c = 0.0;
      wall_of(cfg, node, axis, side, &act, n, &c);
      if (!act) continue;
      for (int a = 0; a < d; ++a) { stage_in[ns][a] = cur[a]; stage_n[ns][a] = n[a]; }
      stage_c[ns] = c;
      ++ns;
      orc_project(d, cur, n, c, cfg->eps, nxt);
      for (int a = 0; a < d; ++a) cur[a] = nxt[a];
    }
  double g[MAXD], gn[MAXD];
  for (int a = 0; a < d; ++a) g[a] = dv_in[a];
  for (int s = ns - 1; s >= 0; --s) {
    orc_project_adj(d, stage_in[s], stage_n[s], stage_c[s], cfg->eps, g, gn);
    for (int a = 0; a < d; ++a) g[a] = gn[a];
  }
  /* g = dL/dvbar; gravity term has unit derivative (R5) */
  double pg = 0.0;
  for (int a = 0; a < d; ++a) {
    dp[a] = g[a] / m;   /* (D) */
    pg += p[a] * g[a];
  }
  *dm = -pg / (m * m); /* (E), first form */
}

/* ------------------------------------------------------------------------------------ */
/* helpers for the stencil                                                              */
/* ------------------------------------------------------------------------------------ */
static int S_of(int d) { return 2 * d + 2 * d * d; }
static int nodes_of(const orc_cfg* cfg) {
  int nn = 1;
  for (int a = 0; a < cfg->dim; ++a) nn *= cfg->res;
  return nn;
}
static int node_index(const orc_cfg* cfg, const int* i) {
  int idx = 0;
  for (int a = 0; a < cfg->dim; ++a) idx = idx * cfg->res + i[a];
  return idx;
}
static int n_stencil(int d) { return d == 2 ? 9 : 27; }
static void stencil_offset(int d, int s, int* o) {
  if (d == 2) { o[0] = s / 3; o[1] = s % 3; }
  else { o[0] = s / 9; o[1] = (s / 3) % 3; o[2] = s % 3; }
}

/* per-particle quantities of step n shared by P2G and the adjoint */
typedef struct {
  int base[MAXD];
  double w[MAXD][3], dw[MAXD][3];
  double mu, lam, J, lnJ;
  double P[9];     /* total PK1: P(F) + F sigma (S1) */
  double Pel[9];   /* elastic part P(F)                     */
  double sigma[9]; /* actuation stress sigma_pa              */
  double G[9];     /* G_p                     */
} pq_t;

static int particle_quantities(const orc_cfg* cfg, const double* rec, double mass, double vol,
                               double E, double nu, int aid, const double* act_t, pq_t* q) {
  int d = cfg->dim;
  double dx = 1.0 / (double)cfg->res;
  const double* x = rec;
  const double* C = rec + 2 * d;
  const double* F = rec + 2 * d + d * d;
  for (int a = 0; a < d; ++a) {
    orc_weights(x[a] / dx, &q->base[a], q->w[a], q->dw[a]);
    if (q->base[a] < 0 || q->base[a] > cfg->res - 3) return ORC_ERR_OUT_OF_DOMAIN; /* R14 */
  }
  q->J = orc_det(d, F);
  if (!(q->J > 0.0)) return ORC_ERR_INVERTED; /* R14 */
  q->lnJ = log(q->J);
  orc_lame(E, nu, &q->mu, &q->lam);
  if (cfg->material == 1) orc_pk1_fcr(d, F, q->mu, q->lam, q->Pel);
  else orc_pk1(d, F, q->mu, q->lam, q->Pel);
  for (int i = 0; i < d * d; ++i) q->sigma[i] = 0.0;
  if (aid >= 0)
    for (int a = 0; a < d; ++a) q->sigma[a * d + a] = cfg->act_strength * act_t[aid * d + a]; /* R4 */
  /* P = P(F) + F sigma   (S1) */
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      double fs = 0.0;
      for (int g = 0; g < d; ++g) fs += F[a * d + g] * q->sigma[g * d + b];
      q->P[a * d + b] = q->Pel[a * d + b] + fs;
    }
  /* G = -(4/dx^2) dt V P F^T + m C   (Eq. 4) */
  double k = 4.0 / (dx * dx) * cfg->dt * vol;
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      double pft = 0.0;
      for (int g = 0; g < d; ++g) pft += q->P[a * d + g] * F[b * d + g];
      q->G[a * d + b] = -k * pft + mass * C[a * d + b];
    }
  return ORC_OK;
}

/* weight W and its x_p-gradient dW[alpha] for stencil offset o (R10: dN/dx_p). */
static void stencil_weight(int d, const pq_t* q, const int* o, double res, double* W,
                           double* dW) {
  double w = 1.0;
  for (int a = 0; a < d; ++a) w *= q->w[a][o[a]];
  *W = w;
  for (int a = 0; a < d; ++a) {
    double g = res * q->dw[a][o[a]];
    for (int b = 0; b < d; ++b)
      if (b != a) g *= q->w[b][o[b]];
    dW[a] = g;
  }
}

/* ------------------------------------------------------------------------------------ */
/* forward: one step, P2G (Eqs. 3-5), grid (Eq. 6 + R5/R6), G2P (Eqs. 7-10)               */
/* ------------------------------------------------------------------------------------ */
typedef struct {
  double* m;    /* [nn]     */
  double* p;    /* [nn][d]  */
  double* vbar; /* [nn][d]  after Eq. 6 and gravity, before projection */
  double* v;    /* [nn][d]  after projection                            */
} grid_t;

/* P2G of one particle (Eqs. 3, 5) into the grid arrays m, p; node ni is stored at
 * m[ni - lo] (lo = 0: the whole grid; the OpenMP timing build scatters a thread's particles
 * into a private sub-range, oracle/mpm_oracle_omp.c). */
static void p2g_particle(const orc_cfg* cfg, const double* rec, double mass, const pq_t* q,
                         double* m, double* p, int lo) {
  int d = cfg->dim, ns = n_stencil(d);
  double dx = 1.0 / (double)cfg->res;
  const double* x = rec;
  const double* v = rec + d;
  for (int s = 0; s < ns; ++s) {
    int o[MAXD], i[MAXD];
    stencil_offset(d, s, o);
    double W = 1.0, dpos[MAXD];
    for (int a = 0; a < d; ++a) {
      i[a] = q->base[a] + o[a];
      W *= orc_N(x[a] / dx - (double)i[a]); /* N(x_i - x_p), R2 */
      dpos[a] = (double)i[a] * dx - x[a];   /* x_i - x_p        */
    }
    int ni = node_index(cfg, i) - lo;
    m[ni] += W * mass; /* Eq. 3 */
    for (int a = 0; a < d; ++a) {
      double Gd = 0.0;
      for (int b = 0; b < d; ++b) Gd += q->G[a * d + b] * dpos[b];
      p[ni * d + a] += W * (mass * v[a] + Gd); /* Eq. 5 */
    }
  }
}

/* the grid operation of node ni (Eq. 6 + R5/R6) */
static void grid_node_at(const orc_cfg* cfg, grid_t* g, int ni) {
  int d = cfg->dim, node[MAXD], r = ni;
  for (int a = d - 1; a >= 0; --a) { node[a] = r % cfg->res; r /= cfg->res; }
  orc_grid_node(cfg, node, g->m[ni], g->p + ni * d, g->vbar + ni * d, g->v + ni * d);
}

static int p2g_and_grid(const orc_cfg* cfg, const double* st, const double* mass,
                        const double* vol, const double* E, const double* nu, const int* act_id,
                        const double* act_t, grid_t* g, pq_t* pq, int* bad) {
  int d = cfg->dim, S = S_of(d), nn = nodes_of(cfg);
  memset(g->m, 0, sizeof(double) * nn);
  memset(g->p, 0, sizeof(double) * nn * d);
  for (int pi = 0; pi < cfg->n; ++pi) {
    const double* rec = st + (size_t)pi * S;
    int err = particle_quantities(cfg, rec, mass[pi], vol[pi], E[pi], nu[pi], act_id[pi],
                                  act_t, &pq[pi]);
    if (err) { *bad = pi; return err; }
    p2g_particle(cfg, rec, mass[pi], &pq[pi], g->m, g->p, 0);
  }
  for (int ni = 0; ni < nn; ++ni) grid_node_at(cfg, g, ni);
  return ORC_OK;
}

/* G2P of particle pi (Eqs. 7-10) */
static void g2p_particle(const orc_cfg* cfg, const double* st, const grid_t* g, const pq_t* pq,
                         double* out, int pi) {
  int d = cfg->dim, S = S_of(d), ns = n_stencil(d);
  double dx = 1.0 / (double)cfg->res;
  {
    const double* rec = st + (size_t)pi * S;
    const double* x = rec;
    const double* F = rec + 2 * d + d * d;
    double vn[MAXD] = {0, 0, 0}, Cn[9] = {0};
    for (int s = 0; s < ns; ++s) {
      int o[MAXD], i[MAXD];
      stencil_offset(d, s, o);
      double W = 1.0, dpos[MAXD];
      for (int a = 0; a < d; ++a) {
        i[a] = pq[pi].base[a] + o[a];
        W *= orc_N(x[a] / dx - (double)i[a]);
        dpos[a] = (double)i[a] * dx - x[a];
      }
      const double* vi = g->v + node_index(cfg, i) * d;
      for (int a = 0; a < d; ++a) {
        vn[a] += W * vi[a]; /* Eq. 7 */
        for (int b = 0; b < d; ++b) Cn[a * d + b] += 4.0 / (dx * dx) * W * vi[a] * dpos[b]; /* Eq. 8 */
      }
    }
    double* o_rec = out + (size_t)pi * S;
    double* xo = o_rec;
    double* vo = o_rec + d;
    double* Co = o_rec + 2 * d;
    double* Fo = o_rec + 2 * d + d * d;
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) {
        double acc = 0.0; /* Eq. 9: F' = (I + dt C') F */
        for (int g2 = 0; g2 < d; ++g2)
          acc += ((a == g2 ? 1.0 : 0.0) + cfg->dt * Cn[a * d + g2]) * F[g2 * d + b];
        Fo[a * d + b] = acc;
        Co[a * d + b] = Cn[a * d + b];
      }
    for (int a = 0; a < d; ++a) {
      vo[a] = vn[a];
      xo[a] = x[a] + cfg->dt * vn[a]; /* Eq. 10 */
    }
  }
}

static void g2p(const orc_cfg* cfg, const double* st, const grid_t* g, const pq_t* pq,
                double* out) {
  for (int pi = 0; pi < cfg->n; ++pi) g2p_particle(cfg, st, g, pq, out, pi);
}

static int alloc_grid(const orc_cfg* cfg, grid_t* g) {
  int nn = nodes_of(cfg), d = cfg->dim;
  g->m = (double*)calloc((size_t)nn, sizeof(double));
  g->p = (double*)calloc((size_t)nn * d, sizeof(double));
  g->vbar = (double*)calloc((size_t)nn * d, sizeof(double));
  g->v = (double*)calloc((size_t)nn * d, sizeof(double));
  return (g->m && g->p && g->vbar && g->v) ? 0 : -1;
}
static void free_grid(grid_t* g) {
  free(g->m); free(g->p); free(g->vbar); free(g->v);
}

static int check_cfg(const orc_cfg* cfg) {
  if (!cfg || (cfg->dim != 2 && cfg->dim != 3) || cfg->res < 8 || cfg->n < 0 || cfg->n_act < 0)
    return ORC_ERR_ARG;
  return ORC_OK;
}

int orc_step_grid(const orc_cfg* cfg, const double* state, const double* mass,
                  const double* vol, const double* E, const double* nu, const int* act_id,
                  const double* act_t, double* m, double* p, double* vbar, double* v) {
  if (check_cfg(cfg)) return ORC_ERR_ARG;
  int nn = nodes_of(cfg), d = cfg->dim;
  grid_t g;
  if (alloc_grid(cfg, &g)) return ORC_ERR_ARG;
  pq_t* pq = (pq_t*)malloc(sizeof(pq_t) * (size_t)(cfg->n > 0 ? cfg->n : 1));
  int bad = -1;
  int err = p2g_and_grid(cfg, state, mass, vol, E, nu, act_id, act_t, &g, pq, &bad);
  if (!err) {
    memcpy(m, g.m, sizeof(double) * nn);
    memcpy(p, g.p, sizeof(double) * nn * d);
    memcpy(vbar, g.vbar, sizeof(double) * nn * d);
    memcpy(v, g.v, sizeof(double) * nn * d);
  }
  free(pq);
  free_grid(&g);
  return err;
}

int orc_forward(const orc_cfg* cfg, int n_steps, double* traj, const double* mass,
                const double* vol, const double* E, const double* nu, const int* act_id,
                const double* act, int* err_index) {
  if (check_cfg(cfg) || n_steps < 0) return ORC_ERR_ARG;
  int d = cfg->dim, S = S_of(d);
  grid_t g;
  if (alloc_grid(cfg, &g)) return ORC_ERR_ARG;
  pq_t* pq = (pq_t*)malloc(sizeof(pq_t) * (size_t)(cfg->n > 0 ? cfg->n : 1));
  int err = ORC_OK;
  for (int t = 0; t < n_steps; ++t) {
    const double* st = traj + (size_t)t * cfg->n * S;
    double* out = traj + (size_t)(t + 1) * cfg->n * S;
    const double* act_t = act ? act + (size_t)t * cfg->n_act * d : NULL;
    int bad = -1;
    err = p2g_and_grid(cfg, st, mass, vol, E, nu, act_id, act_t, &g, pq, &bad);
    if (err) {
      if (err_index) { err_index[0] = t; err_index[1] = bad; }
      break;
    }
    g2p(cfg, st, &g, pq, out);
  }
  free(pq);
  free_grid(&g);
  return err;
}

/* ------------------------------------------------------------------------------------ */
/* backward of one step n: adjoint record of state n+1 -> adjoint record of state n       */
/* ------------------------------------------------------------------------------------ */
/* (C) P:515-521 for particle pi: scatter into dvi (node ni stored at dvi[(ni - lo) d]) */
static void g2pT_particle(const orc_cfg* cfg, const double* st, const pq_t* pq, const double* gvh,
                          const double* gCh, double* dvi, int lo, int pi) {
  int d = cfg->dim, S = S_of(d), ns = n_stencil(d);
  double dx = 1.0 / (double)cfg->res;
  const double* x = st + (size_t)pi * S;
  for (int s = 0; s < ns; ++s) {
    int o[MAXD], i[MAXD];
    stencil_offset(d, s, o);
    double W = 1.0, dpos[MAXD];
    for (int a = 0; a < d; ++a) {
      i[a] = pq[pi].base[a] + o[a];
      W *= orc_N(x[a] / dx - (double)i[a]);
      dpos[a] = (double)i[a] * dx - x[a];
    }
    int ni = node_index(cfg, i) - lo;
    for (int a = 0; a < d; ++a) {
      double cd = 0.0;
      for (int b = 0; b < d; ++b) cd += gCh[(pi * d + a) * d + b] * dpos[b];
      dvi[ni * d + a] += gvh[pi * d + a] * W + 4.0 / (dx * dx) * W * cd;
    }
  }
}

/* (L) P:609-635, (D) P:525-530, (E) P:534-540 of node ni */
static void grid_node_adj_at(const orc_cfg* cfg, const grid_t* g, const double* dvi, double* dpi,
                             double* dmi, int ni) {
  int d = cfg->dim, node[MAXD], r = ni;
  for (int a = d - 1; a >= 0; --a) { node[a] = r % cfg->res; r /= cfg->res; }
  orc_grid_node_adj(cfg, node, g->m[ni], g->p + ni * d, dvi + ni * d, dpi + ni * d, &dmi[ni]);
}

/* (A) P:496-501, (B) P:504-509 of particle pi, with the carry-over note P:511 (gin already
 * holds dL/dv^{n+1}, dL/dC^{n+1} from the later step) */
static void stepAB_particle(const orc_cfg* cfg, const double* st, const double* gin, double* gvh,
                            double* gCh, int pi) {
  int d = cfg->dim, S = S_of(d);
  const double* gr = gin + (size_t)pi * S;
  const double* gx = gr;
  const double* gv = gr + d;
  const double* gC = gr + 2 * d;
  const double* gF = gr + 2 * d + d * d;
  const double* F = st + (size_t)pi * S + 2 * d + d * d;
  for (int a = 0; a < d; ++a) gvh[pi * d + a] = gv[a] + cfg->dt * gx[a];
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      double s = 0.0;
      for (int c = 0; c < d; ++c) s += gF[a * d + c] * F[b * d + c];
      gCh[(pi * d + a) * d + b] = gC[a * d + b] + cfg->dt * s;
    }
}

static void p2gT_particle(const orc_cfg* cfg, const double* st, const double* st_next,
                          const double* mass, const double* vol, const double* E, const double* nu,
                          const int* act_id, const double* gin, double* gout, double* gE, double* gnu,
                          double* ga_t, double* gm, const grid_t* g, const pq_t* pq, const double* gvh,
                          const double* gCh, const double* dpi, const double* dmi, int pi);

static int step_backward(const orc_cfg* cfg, const double* st, const double* st_next,
                         const double* mass, const double* vol, const double* E,
                         const double* nu, const int* act_id, const double* act_t,
                         const double* gin, double* gout, double* gE, double* gnu,
                         double* ga_t, double* gm, grid_t* g, pq_t* pq, double* dvi, double* dpi,
                         double* dmi) {
  int d = cfg->dim, nn = nodes_of(cfg);
  int bad = -1;
  /* recompute step n's grid from the memo */
  int err = p2g_and_grid(cfg, st, mass, vol, E, nu, act_id, act_t, g, pq, &bad);
  if (err) return err;

  double* gvh = (double*)malloc(sizeof(double) * (size_t)(cfg->n > 0 ? cfg->n : 1) * d);
  double* gCh = (double*)malloc(sizeof(double) * (size_t)(cfg->n > 0 ? cfg->n : 1) * d * d);

  /* (A), (B) */
  for (int pi = 0; pi < cfg->n; ++pi) stepAB_particle(cfg, st, gin, gvh, gCh, pi);
  /* (C) P:515-521: scatter to dL/dv_i */
  memset(dvi, 0, sizeof(double) * nn * d);
  for (int pi = 0; pi < cfg->n; ++pi) g2pT_particle(cfg, st, pq, gvh, gCh, dvi, 0, pi);
  /* (L) P:609-635, then (D) P:525-530 and (E) P:534-540 per node */
  for (int ni = 0; ni < nn; ++ni) grid_node_adj_at(cfg, g, dvi, dpi, dmi, ni);
  /* (F)-(K) P:543-605 per particle */
  for (int pi = 0; pi < cfg->n; ++pi)
    p2gT_particle(cfg, st, st_next, mass, vol, E, nu, act_id, gin, gout, gE, gnu, ga_t, gm, g, pq, gvh,
                  gCh, dpi, dmi, pi);
  free(gvh);
  free(gCh);
  return ORC_OK;
}

/* (F)-(K) P:543-605 of particle pi; adds its actuation gradient to ga_t (step K) */
static void p2gT_particle(const orc_cfg* cfg, const double* st, const double* st_next,
                          const double* mass, const double* vol, const double* E, const double* nu,
                          const int* act_id, const double* gin, double* gout, double* gE, double* gnu,
                          double* ga_t, double* gm, const grid_t* g, const pq_t* pq, const double* gvh,
                          const double* gCh, const double* dpi, const double* dmi, int pi) {
  int d = cfg->dim, S = S_of(d), ns = n_stencil(d);
  double dx = 1.0 / (double)cfg->res, res = (double)cfg->res;
  {
    const double* rec = st + (size_t)pi * S;
    const double* x = rec;
    const double* v = rec + d;
    const double* F = rec + 2 * d + d * d;
    const double* Cnext = st_next + (size_t)pi * S + 2 * d;
    const double* gr = gin + (size_t)pi * S;
    const double* gx = gr;
    const double* gF = gr + 2 * d + d * d;
    double* go = gout + (size_t)pi * S;
    double* dx_o = go;
    double* dv_o = go + d;
    double* dC_o = go + 2 * d;
    double* dF_o = go + 2 * d + d * d;
    const pq_t* q = &pq[pi];
    double m = mass[pi];
    double k = 4.0 / (dx * dx) * cfg->dt * vol[pi];
    double dP[9] = {0};
    for (int a = 0; a < d; ++a) { dv_o[a] = 0.0; dx_o[a] = gx[a]; }
    for (int a = 0; a < d * d; ++a) { dC_o[a] = 0.0; dF_o[a] = 0.0; }
    for (int s = 0; s < ns; ++s) {
      int o[MAXD], i[MAXD];
      stencil_offset(d, s, o);
      double W, dW[MAXD], dpos[MAXD];
      for (int a = 0; a < d; ++a) {
        i[a] = q->base[a] + o[a];
        dpos[a] = (double)i[a] * dx - x[a];
      }
      stencil_weight(d, q, o, res, &W, dW);
      int ni = node_index(cfg, i);
      const double* dp = dpi + ni * d;
      const double* vi = g->v + ni * d;
      double dm = dmi[ni];
      for (int a = 0; a < d; ++a) {
        dv_o[a] += W * m * dp[a]; /* (F) P:548 */
        for (int b = 0; b < d; ++b) {
          double fd = 0.0;
          for (int c = 0; c < d; ++c) fd += F[c * d + b] * dpos[c];
          dP[a * d + b] += -W * k * dp[a] * fd;      /* (G) P:557 */
          dC_o[a * d + b] += W * dp[a] * m * dpos[b]; /* (I) P:577 */
        }
      }
      /* last term of (H): through the F^T factor of P F^T, with P the total PK1 */
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
          double s2 = 0.0;
          for (int c = 0; c < d; ++c) s2 += dp[c] * k * q->P[c * d + b];
          dF_o[a * d + b] += -W * s2 * dpos[a];
        }
      /* (J) P:590-596, with dN read as dN/dx_p (R10) */
      for (int a = 0; a < d; ++a) {
        double t2 = 0.0, t3 = 0.0, t4 = 0.0;
        for (int b = 0; b < d; ++b) {
          t2 += gvh[pi * d + b] * dW[a] * vi[b];
          double inner = 0.0;
          for (int c = 0; c < d; ++c) inner += gCh[(pi * d + b) * d + c] * dW[a] * vi[b] * dpos[c];
          t3 += 4.0 / (dx * dx) * (-gCh[(pi * d + b) * d + a] * W * vi[b] + inner);
          double Gd = 0.0;
          for (int c = 0; c < d; ++c) Gd += q->G[b * d + c] * dpos[c];
          t4 += dp[b] * (dW[a] * (m * v[b] + Gd) - W * q->G[b * d + a]);
        }
        double t5 = m * dm * dW[a];
        dx_o[a] += t2 + t3 + t4 + t5;
      }
      /* NEXT N3: dL/dm_p = sum_i N dL/dm_i + sum_i N dL/dp_i . (v_p + C_p (x_i - x_p))
       * (chain rule through Eqs. 3-5; formula as restated in SPEC.md:324) */
      if (gm) {
        const double* Cp = rec + 2 * d;
        double sm = dm;
        for (int a = 0; a < d; ++a) {
          double cd = 0.0;
          for (int b = 0; b < d; ++b) cd += Cp[a * d + b] * dpos[b];
          sm += dp[a] * (v[a] + cd);
        }
        gm[pi] += W * sm;
      }
    }
    /* (H) P:561-568: first three terms */
    double H[81];
    if (cfg->material == 1) orc_dPdF_fcr(d, F, q->mu, q->lam, H);
    else orc_dPdF(d, F, q->mu, q->lam, H);
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) {
        double t1 = 0.0, t2 = 0.0, t3 = 0.0;
        for (int c = 0; c < d; ++c)
          t1 += gF[c * d + b] * ((c == a ? 1.0 : 0.0) + cfg->dt * Cnext[c * d + a]);
        for (int c = 0; c < d; ++c)
          for (int e = 0; e < d; ++e) t2 += dP[c * d + e] * H[((c * d + e) * d + a) * d + b];
        for (int c = 0; c < d; ++c) t3 += dP[a * d + c] * q->sigma[b * d + c];
        dF_o[a * d + b] += t1 + t2 + t3;
      }
    /* (K) P:600-605 (n+1 -> n, R11): dL/dsigma_ab = sum_g dP_gb F_ga ; sigma = s Diag(a) (R4) */
    if (act_id[pi] >= 0 && ga_t) {
      for (int a = 0; a < d; ++a) {
        double dsig = 0.0;
        for (int c = 0; c < d; ++c) dsig += dP[c * d + a] * F[c * d + a];
        ga_t[act_id[pi] * d + a] += cfg->act_strength * dsig;
      }
    }
    /* material parameters (R19): dL/dmu = dP : dP/dmu, dL/dlam = dP : dP/dlam */
    double Fi[9], Rp[9];
    orc_inv(d, F, Fi);
    if (cfg->material == 1) orc_polar(d, F, Rp);
    double dmu = 0.0, dlam = 0.0;
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) {
        double FinvT = Fi[b * d + a];
        if (cfg->material == 1) { /* dP/dmu = 2 (F - R), dP/dlam = (J - 1) J F^-T */
          dmu += dP[a * d + b] * 2.0 * (F[a * d + b] - Rp[a * d + b]);
          dlam += dP[a * d + b] * (q->J - 1.0) * q->J * FinvT;
        } else {
          dmu += dP[a * d + b] * (F[a * d + b] - FinvT);
          dlam += dP[a * d + b] * q->lnJ * FinvT;
        }
      }
    double Ev = E[pi], nv = nu[pi];
    double dmu_dE = 1.0 / (2.0 * (1.0 + nv));
    double dlam_dE = nv / ((1.0 + nv) * (1.0 - 2.0 * nv));
    double dmu_dnu = -Ev / (2.0 * (1.0 + nv) * (1.0 + nv));
    double dlam_dnu = Ev * (1.0 + 2.0 * nv * nv) /
                      ((1.0 + nv) * (1.0 + nv) * (1.0 - 2.0 * nv) * (1.0 - 2.0 * nv));
    gE[pi] += dmu * dmu_dE + dlam * dlam_dE;
    gnu[pi] += dmu * dmu_dnu + dlam * dlam_dnu;
  }
}

int orc_backward_ex(const orc_cfg* cfg, int n_steps, const double* traj, const double* mass,
                    const double* vol, const double* E, const double* nu, const int* act_id,
                    const double* act, const double* seeds, double* grad0, double* gE,
                    double* gnu, double* ga, double* gm) {
  if (check_cfg(cfg) || n_steps < 0) return ORC_ERR_ARG;
  int d = cfg->dim, S = S_of(d), nn = nodes_of(cfg);
  size_t rec = (size_t)cfg->n * S;
  grid_t g;
  if (alloc_grid(cfg, &g)) return ORC_ERR_ARG;
  pq_t* pq = (pq_t*)malloc(sizeof(pq_t) * (size_t)(cfg->n > 0 ? cfg->n : 1));
  double* dvi = (double*)calloc((size_t)nn * d, sizeof(double));
  double* dpi = (double*)calloc((size_t)nn * d, sizeof(double));
  double* dmi = (double*)calloc((size_t)nn, sizeof(double));
  double* a = (double*)malloc(sizeof(double) * (rec > 0 ? rec : 1));
  double* b = (double*)malloc(sizeof(double) * (rec > 0 ? rec : 1));
  /* the adjoint of state T is its own seed; every earlier state t adds seeds[t] (NEXT N4:
   * a running loss sum_t L_t(state_t) -- chain rule of P:165 with per-step terms) */
  memcpy(a, seeds + (size_t)n_steps * rec, sizeof(double) * rec);
  for (int pi = 0; pi < cfg->n; ++pi) { gE[pi] = 0.0; gnu[pi] = 0.0; if (gm) gm[pi] = 0.0; }
  if (ga) memset(ga, 0, sizeof(double) * (size_t)n_steps * cfg->n_act * d);
  int err = ORC_OK;
  for (int t = n_steps - 1; t >= 0; --t) {
    const double* act_t = act ? act + (size_t)t * cfg->n_act * d : NULL;
    double* ga_t = ga ? ga + (size_t)t * cfg->n_act * d : NULL;
    err = step_backward(cfg, traj + (size_t)t * rec, traj + (size_t)(t + 1) * rec, mass, vol, E,
                        nu, act_id, act_t, a, b, gE, gnu, ga_t, gm, &g, pq, dvi, dpi, dmi);
    if (err) break;
    for (size_t q = 0; q < rec; ++q) b[q] += seeds[(size_t)t * rec + q];
    double* tmp = a; a = b; b = tmp;
  }
  if (!err) memcpy(grad0, a, sizeof(double) * rec);
  free(a); free(b); free(dvi); free(dpi); free(dmi); free(pq);
  free_grid(&g);
  return err;
}

int orc_backward(const orc_cfg* cfg, int n_steps, const double* traj, const double* mass,
                 const double* vol, const double* E, const double* nu, const int* act_id,
                 const double* act, const double* seed, double* grad0, double* gE, double* gnu,
                 double* ga) {
  if (check_cfg(cfg) || n_steps < 0) return ORC_ERR_ARG;
  size_t rec = (size_t)cfg->n * S_of(cfg->dim);
  double* seeds = (double*)calloc((size_t)(n_steps + 1) * (rec > 0 ? rec : 1), sizeof(double));
  memcpy(seeds + (size_t)n_steps * rec, seed, sizeof(double) * rec);
  int err = orc_backward_ex(cfg, n_steps, traj, mass, vol, E, nu, act_id, act, seeds, grad0, gE,
                            gnu, ga, NULL);
  free(seeds);
  return err;
}

/* ------------------------------------------------------------------------------------ */
/* Binning (north_star item 1), decided on the fp32 positions (R17):                      */
/*   xg = x * res (fp32, exact for power-of-two res); base = floor(xg - 0.5f) (fp32);      */
/*   block edge Bb = 4 (3D) / 8 (2D); block = base / Bb; cell = base % Bb;                 */
/*   key = (rollout * nb + linear(block)) * Bb^d + linear(cell), row-major, axis 0 slowest */
/*   perm = stable sort of key (ties keep index order); block_start = exclusive prefix.   */
/* ------------------------------------------------------------------------------------ */
typedef struct { int key; int idx; } kv_t;
static int cmp_kv(const void* A, const void* B) {
  const kv_t* a = (const kv_t*)A;
  const kv_t* b = (const kv_t*)B;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx ? 1 : 0);
}

int orc_bin(int dim, int res, int batch, int n, const float* x, int* key, int* perm,
            int* block_start) {
  if ((dim != 2 && dim != 3) || res < 8 || batch < 0 || n < 0) return ORC_ERR_ARG;
  int Bb = dim == 3 ? 4 : 8;
  if (res % Bb) return ORC_ERR_ARG;
  int nbpa = res / Bb, nb = 1, cpb = 1;
  for (int a = 0; a < dim; ++a) { nb *= nbpa; cpb *= Bb; }
  size_t total = (size_t)batch * n;
  kv_t* kv = (kv_t*)malloc(sizeof(kv_t) * (total > 0 ? total : 1));
  for (size_t p = 0; p < total; ++p) {
    int r = (int)(p / (size_t)n);
    int blk = 0, cell = 0;
    for (int a = 0; a < dim; ++a) {
      float xg = x[p * dim + a] * (float)res;
      int base = (int)floorf(xg - 0.5f);
      if (base < 0 || base > res - 3) { free(kv); return ORC_ERR_OUT_OF_DOMAIN; }
      blk = blk * nbpa + base / Bb;
      cell = cell * Bb + base % Bb;
    }
    kv[p].key = (r * nb + blk) * cpb + cell;
    kv[p].idx = (int)p;
    key[p] = kv[p].key;
  }
  qsort(kv, total, sizeof(kv_t), cmp_kv);
  for (size_t s = 0; s < total; ++s) perm[s] = kv[s].idx;
  /* block_start[g] = number of particles whose key / cpb < g */
  size_t nblk = (size_t)batch * nb;
  size_t s = 0;
  for (size_t gb = 0; gb <= nblk; ++gb) {
    while (s < total && (size_t)(kv[s].key / cpb) < gb) ++s;
    block_start[gb] = (int)s;
  }
  free(kv);
  return ORC_OK;
}
