/*
 * mpm_oracle_omp.c -- OpenMP timing build of the CPU oracle ("an OpenMP
 * variant at os.cpu_count() threads, with per-thread grids merged in fixed order").
 *
 * TEST / MEASUREMENT INFRASTRUCTURE ONLY: bench.py's cpu_baseline leg times it; the tests
 * check it against the serial oracle (tests/test_oracle_omp.py).  It adds no arithmetic of
 * the method: it includes mpm_oracle.c and calls the same per-particle and per-node
 * functions (p2g_particle, grid_node_at, g2p_particle, stepAB_particle, g2pT_particle,
 * grid_node_adj_at, p2gT_particle) from parallel loops.  The two scatters (P2G, step C) go
 * into per-chunk private grids -- chunk c = the contiguous particles [n c / T, n (c+1) / T),
 * each covering the node-index range its stencils touch -- and the chunk grids are summed in
 * chunk order (deterministic for a given T; equal to the serial oracle up to the summation
 * order of the node sums).  The step-K actuation sums are per-chunk arrays merged in chunk
 * order.  Everything else is per particle or per node.
 *
 * Built by oracle.build_omp() with -fopenmp (fp64), and with -Ddouble=float
 * -fsingle-precision-constant -include tgmath.h for the fp32 timing variant.
 */
#include "mpm_oracle.c"

#include <omp.h>

typedef struct {
  int lo, hi;   /* node-index range [lo, hi] of the chunk's stencils */
  double* m;    /* [hi - lo + 1]      */
  double* p;    /* [hi - lo + 1][d]   (P2G) or dL/dv_i (step C) */
} chunk_grid_t;

static void chunk_bounds(const orc_cfg* cfg, const pq_t* pq, int c, int T, int* p0, int* p1, int* lo,
                         int* hi) {
  int d = cfg->dim;
  *p0 = (int)((long long)cfg->n * c / T);
  *p1 = (int)((long long)cfg->n * (c + 1) / T);
  int l = 0x7fffffff, h = -1;
  for (int pi = *p0; pi < *p1; ++pi) {
    int i0[MAXD], i2[MAXD];
    for (int a = 0; a < d; ++a) { i0[a] = pq[pi].base[a]; i2[a] = pq[pi].base[a] + 2; }
    int a0 = node_index(cfg, i0), a2 = node_index(cfg, i2);
    if (a0 < l) l = a0;
    if (a2 > h) h = a2;
  }
  *lo = l;
  *hi = h;
}

/* scatter of every particle into per-chunk grids, then the fixed-order merge into (m, p);
 * m may be NULL (step C: only the vector part) */
static void scatter_chunks(const orc_cfg* cfg, const pq_t* pq, int T, double* m, double* p,
                           void (*body)(const orc_cfg*, int, double*, double*, int, void*), void* ctx) {
  int d = cfg->dim, nn = nodes_of(cfg);
  chunk_grid_t* ch = (chunk_grid_t*)calloc((size_t)T, sizeof(chunk_grid_t));
#pragma omp parallel for schedule(static, 1)
  for (int c = 0; c < T; ++c) {
    int p0, p1;
    chunk_bounds(cfg, pq, c, T, &p0, &p1, &ch[c].lo, &ch[c].hi);
    if (p1 <= p0) continue;
    size_t len = (size_t)(ch[c].hi - ch[c].lo + 1);
    ch[c].m = m ? (double*)calloc(len, sizeof(double)) : NULL;
    ch[c].p = (double*)calloc(len * d, sizeof(double));
    for (int pi = p0; pi < p1; ++pi) body(cfg, pi, ch[c].m, ch[c].p, ch[c].lo, ctx);
  }
#pragma omp parallel for schedule(static)
  for (int ni = 0; ni < nn; ++ni) {
    double sm = 0.0, sp[MAXD] = {0, 0, 0};
    for (int c = 0; c < T; ++c) {
      if (!ch[c].p || ni < ch[c].lo || ni > ch[c].hi) continue;
      int k = ni - ch[c].lo;
      if (m) sm += ch[c].m[k];
      for (int a = 0; a < d; ++a) sp[a] += ch[c].p[k * d + a];
    }
    if (m) m[ni] = sm;
    for (int a = 0; a < d; ++a) p[ni * d + a] = sp[a];
  }
  for (int c = 0; c < T; ++c) { free(ch[c].m); free(ch[c].p); }
  free(ch);
}

typedef struct {
  const double* st;
  const double* mass;
  const pq_t* pq;
  const double* gvh;
  const double* gCh;
} scat_ctx_t;

static void body_p2g(const orc_cfg* cfg, int pi, double* m, double* p, int lo, void* vctx) {
  const scat_ctx_t* c = (const scat_ctx_t*)vctx;
  p2g_particle(cfg, c->st + (size_t)pi * S_of(cfg->dim), c->mass[pi], &c->pq[pi], m, p, lo);
}

static void body_g2pT(const orc_cfg* cfg, int pi, double* m, double* p, int lo, void* vctx) {
  (void)m;
  const scat_ctx_t* c = (const scat_ctx_t*)vctx;
  g2pT_particle(cfg, c->st, c->pq, c->gvh, c->gCh, p, lo, pi);
}

static int p2g_and_grid_omp(const orc_cfg* cfg, const double* st, const double* mass, const double* vol,
                            const double* E, const double* nu, const int* act_id, const double* act_t,
                            grid_t* g, pq_t* pq, int* bad, int T) {
  int S = S_of(cfg->dim), nn = nodes_of(cfg), err = ORC_OK, first = cfg->n;
#pragma omp parallel for schedule(static) reduction(min : first)
  for (int pi = 0; pi < cfg->n; ++pi)
    if (particle_quantities(cfg, st + (size_t)pi * S, mass[pi], vol[pi], E[pi], nu[pi], act_id[pi], act_t,
                            &pq[pi]) != ORC_OK && pi < first)
      first = pi;
  if (first < cfg->n) {  /* the serial oracle's error: the first failing particle */
    *bad = first;
    return particle_quantities(cfg, st + (size_t)first * S, mass[first], vol[first], E[first], nu[first],
                               act_id[first], act_t, &pq[first]);
  }
  scat_ctx_t ctx = {st, mass, pq, NULL, NULL};
  scatter_chunks(cfg, pq, T, g->m, g->p, body_p2g, &ctx);
#pragma omp parallel for schedule(static)
  for (int ni = 0; ni < nn; ++ni) grid_node_at(cfg, g, ni);
  return err;
}

int orc_omp_threads(void) { return omp_get_max_threads(); }

int orc_forward_omp(const orc_cfg* cfg, int n_steps, double* traj, const double* mass, const double* vol,
                    const double* E, const double* nu, const int* act_id, const double* act, int* err_index) {
  if (check_cfg(cfg) || n_steps < 0) return ORC_ERR_ARG;
  int d = cfg->dim, S = S_of(d), T = omp_get_max_threads();
  grid_t g;
  if (alloc_grid(cfg, &g)) return ORC_ERR_ARG;
  pq_t* pq = (pq_t*)malloc(sizeof(pq_t) * (size_t)(cfg->n > 0 ? cfg->n : 1));
  int err = ORC_OK;
  for (int t = 0; t < n_steps; ++t) {
    const double* st = traj + (size_t)t * cfg->n * S;
    double* out = traj + (size_t)(t + 1) * cfg->n * S;
    const double* act_t = act ? act + (size_t)t * cfg->n_act * d : NULL;
    int bad = -1;
    err = p2g_and_grid_omp(cfg, st, mass, vol, E, nu, act_id, act_t, &g, pq, &bad, T);
    if (err) {
      if (err_index) { err_index[0] = t; err_index[1] = bad; }
      break;
    }
#pragma omp parallel for schedule(static)
    for (int pi = 0; pi < cfg->n; ++pi) g2p_particle(cfg, st, &g, pq, out, pi);
  }
  free(pq);
  free_grid(&g);
  return err;
}

int orc_backward_omp(const orc_cfg* cfg, int n_steps, const double* traj, const double* mass,
                     const double* vol, const double* E, const double* nu, const int* act_id,
                     const double* act, const double* seed, double* grad0, double* gE, double* gnu,
                     double* ga) {
  if (check_cfg(cfg) || n_steps < 0) return ORC_ERR_ARG;
  int d = cfg->dim, S = S_of(d), nn = nodes_of(cfg), T = omp_get_max_threads(), KD = cfg->n_act * d;
  size_t rec = (size_t)cfg->n * S;
  grid_t g;
  if (alloc_grid(cfg, &g)) return ORC_ERR_ARG;
  size_t np = (size_t)(cfg->n > 0 ? cfg->n : 1);
  pq_t* pq = (pq_t*)malloc(sizeof(pq_t) * np);
  double* dvi = (double*)calloc((size_t)nn * d, sizeof(double));
  double* dpi = (double*)calloc((size_t)nn * d, sizeof(double));
  double* dmi = (double*)calloc((size_t)nn, sizeof(double));
  double* a = (double*)malloc(sizeof(double) * (rec > 0 ? rec : 1));
  double* b = (double*)malloc(sizeof(double) * (rec > 0 ? rec : 1));
  double* gvh = (double*)malloc(sizeof(double) * np * d);
  double* gCh = (double*)malloc(sizeof(double) * np * d * d);
  double* ga_c = (double*)calloc((size_t)T * (KD > 0 ? KD : 1), sizeof(double));
  memcpy(a, seed, sizeof(double) * rec);
  for (int pi = 0; pi < cfg->n; ++pi) { gE[pi] = 0.0; gnu[pi] = 0.0; }
  if (ga) memset(ga, 0, sizeof(double) * (size_t)n_steps * KD);
  int err = ORC_OK;
  for (int t = n_steps - 1; t >= 0; --t) {
    const double* st = traj + (size_t)t * rec;
    const double* st_next = traj + (size_t)(t + 1) * rec;
    const double* act_t = act ? act + (size_t)t * KD : NULL;
    int bad = -1;
    err = p2g_and_grid_omp(cfg, st, mass, vol, E, nu, act_id, act_t, &g, pq, &bad, T);
    if (err) break;
#pragma omp parallel for schedule(static)
    for (int pi = 0; pi < cfg->n; ++pi) stepAB_particle(cfg, st, a, gvh, gCh, pi);
    scat_ctx_t ctx = {st, mass, pq, gvh, gCh};
    scatter_chunks(cfg, pq, T, NULL, dvi, body_g2pT, &ctx);
#pragma omp parallel for schedule(static)
    for (int ni = 0; ni < nn; ++ni) grid_node_adj_at(cfg, &g, dvi, dpi, dmi, ni);
    memset(ga_c, 0, sizeof(double) * (size_t)T * (KD > 0 ? KD : 1));
#pragma omp parallel for schedule(static, 1)
    for (int c = 0; c < T; ++c) {
      int p0 = (int)((long long)cfg->n * c / T), p1 = (int)((long long)cfg->n * (c + 1) / T);
      for (int pi = p0; pi < p1; ++pi)
        p2gT_particle(cfg, st, st_next, mass, vol, E, nu, act_id, a, b, gE, gnu, ga ? ga_c + (size_t)c * KD : NULL,
                      NULL, &g, pq, gvh, gCh, dpi, dmi, pi);
    }
    if (ga)
      for (int c = 0; c < T; ++c)
        for (int k = 0; k < KD; ++k) ga[(size_t)t * KD + k] += ga_c[(size_t)c * KD + k];
    double* tmp = a; a = b; b = tmp;
  }
  if (!err) memcpy(grad0, a, sizeof(double) * rec);
  free(a); free(b); free(dvi); free(dpi); free(dmi); free(pq); free(gvh); free(gCh); free(ga_c);
  free_grid(&g);
  return err;
}
