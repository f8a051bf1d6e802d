"""Mutation check of the oracle's pins.

Each mutation is one plausible single-line mistake in oracle/mpm_oracle.c -- a dropped term,
a flipped sign, a transposed operand, a wrong wall / friction mapping -- at one step of the
paper's method.  For every mutation the script builds the mutated file into a temporary
library, points the oracle's loader at it (MPM_ORACLE_LIB) and runs the CPU pins
(tests/test_oracle_*.py, -x).  A mutation is CAUGHT when some pin fails.  Prints one JSON line
per mutation and a summary; exit status 1 if any mutation survives.

    python tools/mutation_check.py [--only NAME] > profiles/r02_mutation_check.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "mpm_oracle.c")

# (name, passage, exact source text, replacement) -- the text must occur in mpm_oracle.c;
# only its first occurrence is mutated
MUTATIONS = [
    ("eq3_mass_weight_dropped", "Eq. 3, P:135",
     "g->m[ni] += W * mass[pi];", "g->m[ni] += mass[pi];"),
    ("eq5_affine_sign", "Eq. 5, P:137",
     "g->p[ni * d + a] += W * (mass[pi] * v[a] + Gd);", "g->p[ni * d + a] += W * (mass[pi] * v[a] - Gd);"),
    ("eq4_C_transposed", "Eq. 4, P:136",
     "q->G[a * d + b] = -k * pft + mass * C[a * d + b];", "q->G[a * d + b] = -k * pft + mass * C[b * d + a];"),
    ("eq4_stress_sign", "Eq. 4, P:136",
     "q->G[a * d + b] = -k * pft + mass * C[a * d + b];", "q->G[a * d + b] = k * pft + mass * C[a * d + b];"),
    ("pk1_lambda_term_dropped", "R1 (P:102-103)",
     "P[a * dim + b] = mu * (F[a * dim + b] - FinvT_ab) + lam * lnJ * FinvT_ab;",
     "P[a * dim + b] = mu * (F[a * dim + b] - FinvT_ab);"),
    ("s1_actuation_F_transposed", "S1, P:430",
     "fs += F[a * d + g] * q->sigma[g * d + b];", "fs += F[g * d + a] * q->sigma[g * d + b];"),
    ("eq8_affine_transposed", "Eq. 8, P:150",
     "Cn[a * d + b] += 4.0 / (dx * dx) * W * vi[a] * dpos[b];",
     "Cn[a * d + b] += 4.0 / (dx * dx) * W * vi[b] * dpos[a];"),
    ("eq9_C_transposed", "Eq. 9, P:151",
     "acc += ((a == g2 ? 1.0 : 0.0) + cfg->dt * Cn[a * d + g2]) * F[g2 * d + b];",
     "acc += ((a == g2 ? 1.0 : 0.0) + cfg->dt * Cn[g2 * d + a]) * F[g2 * d + b];"),
    ("eq10_advection_dropped", "Eq. 10, P:152",
     "xo[a] = x[a] + cfg->dt * vn[a];", "xo[a] = x[a];"),
    ("stepA_dt_term_dropped", "step A, P:496-501",
     "gvh[pi * d + a] = gv[a] + cfg->dt * gx[a];", "gvh[pi * d + a] = gv[a];"),
    ("stepB_F_transposed", "step B, P:504-509",
     "s += gF[a * d + c] * F[b * d + c];", "s += gF[a * d + c] * F[c * d + b];"),
    ("stepC_affine_sign", "step C, P:515-521",
     "dvi[ni * d + a] += gvh[pi * d + a] * W + 4.0 / (dx * dx) * W * cd;",
     "dvi[ni * d + a] += gvh[pi * d + a] * W - 4.0 / (dx * dx) * W * cd;"),
    ("stepE_sign", "step E, P:534-540",
     "*dm = -pg / (m * m);", "*dm = pg / (m * m);"),
    ("stepG_sign", "step G, P:553-558",
     "dP[a * d + b] += -W * k * dp[a] * fd;", "dP[a * d + b] += W * k * dp[a] * fd;"),
    ("stepH_Cnext_transposed", "step H, P:561-569",
     "t1 += gF[c * d + b] * ((c == a ? 1.0 : 0.0) + cfg->dt * Cnext[c * d + a]);",
     "t1 += gF[c * d + b] * ((c == a ? 1.0 : 0.0) + cfg->dt * Cnext[a * d + c]);"),
    ("stepH_sigma_term_sign", "step H, P:567",
     "t3 += dP[a * d + c] * q->sigma[b * d + c];", "t3 -= dP[a * d + c] * q->sigma[b * d + c];"),
    ("stepH_PFt_term_dropped", "step H, P:568",
     "dF_o[a * d + b] += -W * s2 * dpos[a];", "dF_o[a * d + b] += 0.0 * s2 * dpos[a];"),
    ("hessian_sign", "step H psi-Hessian, P:567",
     "v += (mu - lam * lnJ) * Fi[e * d + a] * Fi[b * d + g];",
     "v += (mu + lam * lnJ) * Fi[e * d + a] * Fi[b * d + g];"),
    ("stepI_transposed", "step I, P:573-578",
     "dC_o[a * d + b] += W * dp[a] * m * dpos[b];", "dC_o[a * d + b] += W * dp[b] * m * dpos[a];"),
    ("stepJ_G_transposed", "step J, P:590-596",
     "t4 += dp[b] * (dW[a] * (m * v[b] + Gd) - W * q->G[b * d + a]);",
     "t4 += dp[b] * (dW[a] * (m * v[b] + Gd) - W * q->G[a * d + b]);"),
    ("stepJ_mass_term_dropped", "step J, P:596",
     "double t5 = m * dm * dW[a];", "double t5 = 0.0 * dm * dW[a];"),
    ("stepJ_gC_sign", "step J, P:593",
     "t3 += 4.0 / (dx * dx) * (-gCh[(pi * d + b) * d + a] * W * vi[b] + inner);",
     "t3 += 4.0 / (dx * dx) * (gCh[(pi * d + b) * d + a] * W * vi[b] + inner);"),
    ("stepK_transposed", "step K, P:600-605",
     "for (int c = 0; c < d; ++c) dsig += dP[c * d + a] * F[c * d + a];",
     "for (int c = 0; c < d; ++c) dsig += dP[a * d + c] * F[c * d + a];"),
    ("stepL_R_uses_max", "step L, P:621 (R12)",
     "double R = lt + c * fmin(ln, 0.0);                                                /* P:621 */",
     "double R = lt + c * fmax(ln, 0.0);                                                /* P:621 */"),
    ("stepL_adjoint_friction_sign", "step L adjoint, P:632",
     "dln += dlts * HR * c * Hmln;", "dln -= dlts * HR * c * Hmln;"),
    ("stepL_sticky_ignored", "R6 sticky walls",
     "if (c < 0.0) { /* sticky wall (R6) */", "if (c < -2.0) { /* sticky wall (R6) */"),
    ("wall_low_friction_from_high_wall", "R6 wall bands",
     "*c = cfg->friction[2 * axis];", "*c = cfg->friction[2 * axis + 1];"),
    ("wall_high_normal_sign", "R6 wall bands",
     "n[axis] = -1.0;", "n[axis] = 1.0;"),
    ("corner_axis_order_reversed", "R6 corner order",
     "  for (int axis = 0; axis < d; ++axis)\n    for (int side = 0; side < 2; ++side) {\n      int act;\n      double n[MAXD], c = 0.0;\n      wall_of(cfg, node, axis, side, &act, n, &c);\n      if (!act) continue;\n      orc_project(",
     "  for (int axis = d - 1; axis >= 0; --axis)\n    for (int side = 0; side < 2; ++side) {\n      int act;\n      double n[MAXD], c = 0.0;\n      wall_of(cfg, node, axis, side, &act, n, &c);\n      if (!act) continue;\n      orc_project("),
    ("r19_dnu_sign", "R19 (E, nu chain rule)",
     "double dlam_dnu = Ev * (1.0 + 2.0 * nv * nv) /", "double dlam_dnu = Ev * (1.0 - 2.0 * nv * nv) /"),
    ("n3_mass_grad_affine_dropped", "N3 dL/dm_p (chain rule through Eqs. 3-5)",
     "sm += dp[a] * (v[a] + cd);", "sm += dp[a] * v[a];"),
    ("bspline_inner_piece", "R2 quadratic B-spline",
     "if (a < 0.5) return 0.75 - a * a;", "if (a < 0.5) return 0.75 - 0.5 * a * a;"),
    ("bspline_derivative_sign", "R2 (dN for step J)",
     "if (a < 1.5) return -(1.5 - a) * s;", "if (a < 1.5) return (1.5 - a) * s;"),
    ("binning_cell_index", "R17 binning key",
     "cell = cell * Bb + base % Bb;", "cell = cell * Bb + base / Bb;"),
    ("fcr_pk1_rotation_dropped", "R21 fixed-corotated P",
     "P[a * dim + b] = 2.0 * mu * (F[a * dim + b] - R[a * dim + b]) + lam * (J - 1.0) * J * Fi[b * dim + a];",
     "P[a * dim + b] = 2.0 * mu * F[a * dim + b] + lam * (J - 1.0) * J * Fi[b * dim + a];"),
]

PINS = ["tests/test_oracle_units.py", "tests/test_oracle_step.py", "tests/test_oracle_grad.py",
        "tests/test_oracle_fcr.py", "tests/test_oracle_controller.py"]


def run_one(name, old, new, tmp):
    src = open(SRC).read()
    if old not in src:
        return {"mutation": name, "error": "source text not found"}
    mutated = src.replace(old, new, 1)
    csrc = os.path.join(tmp, f"{name}.c")
    lib = os.path.join(tmp, f"lib_{name}.so")
    with open(csrc, "w") as f:
        f.write(mutated)
    subprocess.check_call(["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                           "-I", os.path.join(ROOT, "oracle"), "-o", lib, csrc, "-lm"])
    env = dict(os.environ, MPM_ORACLE_LIB=lib)
    t0 = time.time()
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "-m", "not gpu", *PINS],
                       cwd=ROOT, env=env, capture_output=True, text=True)
    failed = [ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED ")]
    return {"mutation": name, "caught": r.returncode != 0, "first_failing_pin": failed[0] if failed else None,
            "seconds": round(time.time() - t0, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    caught = 0
    n = 0
    with tempfile.TemporaryDirectory() as tmp:
        for name, cite, old, new in MUTATIONS:
            if args.only and args.only != name:
                continue
            res = run_one(name, old, new, tmp)
            res["passage"] = cite
            print(json.dumps(res), flush=True)
            n += 1
            caught += bool(res.get("caught"))
    print(json.dumps({"summary": f"{caught}/{n} mutations caught by the oracle pins"}), flush=True)
    return 0 if caught == n else 1


if __name__ == "__main__":
    sys.exit(main())
