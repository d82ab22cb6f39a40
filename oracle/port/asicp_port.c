/*
 * asicp_port.c — plain-C restatement of graspmatch::optimize_grasp.
 *
 * TEST INFRASTRUCTURE ONLY (the parity checker; never linked into the
 * product).  A line-by-line CPU restatement of the reference hot path on the
 * POD structs of include/asicp.h, so the checker exists even where the
 * reference sources (and therefore oracle/_ref) are absent.  Every function
 * cites the reference lines it follows; arithmetic is evaluated in the same
 * order as the reference compiled against oracle/shim/Eigen (left-to-right
 * reductions, no FMA: build with -ffp-contract=off), and exp()/log()/pow()/
 * fmod() come from the same libm, so results are bit-identical to the
 * reference (pinned in tests/test_oracle.py against oracle/_ref and the
 * committed golden vectors).
 *
 * Differences in mechanism only: the exact kd-tree nearest neighbour
 * (spatial_index.cpp:14-105) is replaced by an exhaustive scan with the same
 * "strictly closer wins, equal distance -> lowest index" rule
 * (spatial_index.cpp:70, 83), which returns the identical index; the
 * std::thread fan-out (parallel.hpp) is a serial loop (results are
 * worker-count invariant, test_acceptance.cpp:659-680).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "asicp.h"

typedef struct { double x, y, z; } v3;
typedef struct { double m[9]; } m3;

static v3 vadd(v3 a, v3 b) { v3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static v3 vsub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static double vsq(v3 a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }
static double vdot(v3 a, v3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
static v3 vload(const double* p, int64_t i) { v3 r = {p[3 * i], p[3 * i + 1], p[3 * i + 2]}; return r; }
static v3 mmul(const m3* r, v3 p) {
  v3 o = {(r->m[0] * p.x + r->m[1] * p.y) + r->m[2] * p.z, (r->m[3] * p.x + r->m[4] * p.y) + r->m[5] * p.z,
          (r->m[6] * p.x + r->m[7] * p.y) + r->m[8] * p.z};
  return o;
}
static double qsq(const double* q) { return ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]; }

/* geometry.cpp:8-21 */
static m3 rotation_matrix(const double* q) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  m3 r;
  r.m[0] = w * w + x * x - y * y - z * z;
  r.m[1] = 2.0 * (x * y - w * z);
  r.m[2] = 2.0 * (x * z + w * y);
  r.m[3] = 2.0 * (x * y + w * z);
  r.m[4] = w * w - x * x + y * y - z * z;
  r.m[5] = 2.0 * (y * z - w * x);
  r.m[6] = 2.0 * (x * z - w * y);
  r.m[7] = 2.0 * (y * z + w * x);
  r.m[8] = w * w - x * x - y * y + z * z;
  const double n2 = qsq(q);
  for (int i = 0; i < 9; ++i) r.m[i] = r.m[i] / n2;
  return r;
}

/* geometry.cpp:23-32 */
static void rotation_derivatives(const double* q, m3 d[4]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double a[4][9] = {{w, -z, y, z, w, -x, -y, x, w},
                          {x, y, z, y, -x, -w, z, w, -x},
                          {-y, x, w, x, y, z, -w, z, -y},
                          {-z, -w, x, w, -z, y, x, y, z}};
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 9; ++i) d[j].m[i] = a[j][i] * 2.0;
}

/* geometry.cpp:234 */
static void normalize4(double* q) {
  const double n = sqrt(qsq(q));
  for (int i = 0; i < 4; ++i) q[i] = q[i] / n;
}

/* sdf.cpp:177-203 */
static double sdf_query(const asicp_sdf_grid* g, v3 pv) {
  const double p[3] = {pv.x, pv.y, pv.z};
  double hi[3];
  for (int a = 0; a < 3; ++a) hi[a] = g->origin[a] + g->voxel * (double)(g->dims[a] - 1);
  if (p[0] < g->origin[0] || p[1] < g->origin[1] || p[2] < g->origin[2] || p[0] > hi[0] || p[1] > hi[1] ||
      p[2] > hi[2]) {
    double d[3];
    for (int a = 0; a < 3; ++a) {
      double c = p[a] < g->origin[a] ? g->origin[a] : p[a];
      c = hi[a] < c ? hi[a] : c;
      d[a] = p[a] - c;
    }
    return -(sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]) + g->boundary_max_abs);
  }
  double l[3];
  for (int a = 0; a < 3; ++a) l[a] = (p[a] - g->origin[a]) / g->voxel;
  int ix = (int)l[0], iy = (int)l[1], iz = (int)l[2];
  ix = ix < g->dims[0] - 2 ? ix : g->dims[0] - 2;
  iy = iy < g->dims[1] - 2 ? iy : g->dims[1] - 2;
  iz = iz < g->dims[2] - 2 ? iz : g->dims[2] - 2;
  ix = ix > 0 ? ix : 0;
  iy = iy > 0 ? iy : 0;
  iz = iz > 0 ? iz : 0;
#define CL(v) ((v) < 0.0 ? 0.0 : (1.0 < (v) ? 1.0 : (v)))
  const double fx = CL(l[0] - ix), fy = CL(l[1] - iy), fz = CL(l[2] - iz);
#undef CL
  const int ny = g->dims[1], nz = g->dims[2];
#define V(dx, dy, dz) ((double)g->values[((int64_t)(ix + (dx)) * ny + (iy + (dy))) * nz + (iz + (dz))])
  const double c00 = V(0, 0, 0) * (1 - fx) + V(1, 0, 0) * fx;
  const double c01 = V(0, 0, 1) * (1 - fx) + V(1, 0, 1) * fx;
  const double c10 = V(0, 1, 0) * (1 - fx) + V(1, 1, 0) * fx;
  const double c11 = V(0, 1, 1) * (1 - fx) + V(1, 1, 1) * fx;
#undef V
  const double c0 = c00 * (1 - fy) + c10 * fy;
  const double c1 = c01 * (1 - fy) + c11 * fy;
  return c0 * (1 - fz) + c1 * fz;
}

/* sdf.cpp:227-243 colliding_points: fills idx (scene indices), returns count */
static int64_t colliding_points(const asicp_problem* P, const asicp_sdf_grid* g, const double* th, int64_t* idx) {
  double qi[4] = {th[3], -th[4], -th[5], -th[6]};
  const m3 ri = rotation_matrix(qi);
  const v3 t = {th[0], th[1], th[2]};
  v3 ti = mmul(&ri, t);
  ti.x = -ti.x;
  ti.y = -ti.y;
  ti.z = -ti.z;
  const v3 off = {g->offset[0], g->offset[1], g->offset[2]};
  int64_t n = 0;
  for (int64_t c = 0; c < P->n_scene; ++c) {
    const v3 p = vload(P->scene_cloud, c);
    const v3 local = vadd(vadd(mmul(&ri, p), ti), off);
    if (sdf_query(g, vsub(local, off)) > P->contact_tolerance) idx[n++] = c;
  }
  return n;
}

/* Exhaustive nearest neighbour with the kd-tree's tie rule (spatial_index.cpp:63-105). */
static int64_t nearest(const double* pts, const int64_t* map, int64_t n, v3 q) {
  double best = INFINITY;
  int64_t bi = -1;
  for (int64_t i = 0; i < n; ++i) {
    const v3 p = vload(pts, map ? map[i] : i);
    const double d2 = vsq(vsub(p, q));
    if (d2 < best || (d2 == best && i < bi)) {
      best = d2;
      bi = i;
    }
  }
  return bi;
}

/* std::mt19937_64 + Rng::uniform_index (rng.hpp:16-44) */
typedef struct { uint64_t s[312]; int i; } mt64;
static void mt_seed(mt64* m, uint64_t seed) {
  m->s[0] = seed;
  for (int i = 1; i < 312; ++i) m->s[i] = 6364136223846793005ull * (m->s[i - 1] ^ (m->s[i - 1] >> 62)) + (uint64_t)i;
  m->i = 312;
}
static uint64_t mt_next(mt64* m) {
  if (m->i >= 312) {
    static const uint64_t up = 0xFFFFFFFF80000000ull, lo = 0x7FFFFFFFull, a = 0xB5026F5AA96619E9ull;
    int k = 0;
    for (; k < 156; ++k) {
      const uint64_t y = (m->s[k] & up) | (m->s[k + 1] & lo);
      m->s[k] = m->s[k + 156] ^ (y >> 1) ^ ((y & 1) ? a : 0);
    }
    for (; k < 311; ++k) {
      const uint64_t y = (m->s[k] & up) | (m->s[k + 1] & lo);
      m->s[k] = m->s[k - 156] ^ (y >> 1) ^ ((y & 1) ? a : 0);
    }
    const uint64_t y = (m->s[311] & up) | (m->s[0] & lo);
    m->s[311] = m->s[155] ^ (y >> 1) ^ ((y & 1) ? a : 0);
    m->i = 0;
  }
  uint64_t y = m->s[m->i++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}
static uint64_t uniform_index(mt64* m, uint64_t n) {
  unsigned __int128 p = (unsigned __int128)mt_next(m) * n;
  uint64_t l = (uint64_t)p;
  if (l < n) {
    const uint64_t threshold = (0ull - n) % n;
    while (l < threshold) {
      p = (unsigned __int128)mt_next(m) * n;
      l = (uint64_t)p;
    }
  }
  return (uint64_t)(p >> 64);
}

/* spatial_index.cpp:133-139 */
static int64_t minibatch_schedule(int64_t k, int64_t k_max, int64_t n) {
  const double sat = 2.0 * (double)k_max / 3.0;
  const double ramp = ((double)k < sat ? (double)k : sat) / sat;
  int64_t m = llround((double)n * ramp);
  return m < 1 ? 1 : (m > n ? n : m);
}

typedef struct {
  double th[7], loss, prev_loss, grad[7], prior[7];
  int in_col, converged, pre;
} particle;

static void set_err(char* err, size_t len, const char* msg) {
  if (err && len) {
    strncpy(err, msg, len - 1);
    err[len - 1] = 0;
  }
}

/* Evaluate one particle (grasp.cpp:166-194). */
static void evaluate(const asicp_problem* P, particle* pt, mt64* rng, int64_t m, int64_t* colbuf, int64_t* idxbuf,
                     int64_t* pool, double* sw) {
  const asicp_preshape* ps = &P->preshapes[pt->pre];
  const asicp_sdf_grid* g = &P->sdf_grids[ps->sdf_index];
  const int64_t ncol = colliding_points(P, g, pt->th, colbuf);
  const m3 r = rotation_matrix(pt->th + 3);
  const v3 t = {pt->th[0], pt->th[1], pt->th[2]};
  for (int64_t i = 0; i < ps->n_surface; ++i) {
    const v3 w = vadd(mmul(&r, vload(ps->inner_surface, i)), t);
    sw[3 * i] = w.x;
    sw[3 * i + 1] = w.y;
    sw[3 * i + 2] = w.z;
  }
  m3 dR[4];
  rotation_derivatives(pt->th + 3, dR);
  double gt[3] = {0, 0, 0}, gq[4] = {0, 0, 0, 0}, sum = 0.0, mdiv;
  if (ncol > 0) {
    /* collision_loss_and_gradients (grasp.cpp:68-84) + sgd_icp_gradients (optim.cpp:92-106) */
    for (int64_t c = 0; c < ncol; ++c) {
      const v3 rc = vload(P->scene_cloud, colbuf[c]);
      const int64_t nn = nearest(sw, NULL, ps->n_surface, rc);
      const v3 res = vsub(vload(sw, nn), rc);
      sum += vsq(res);
      gt[0] = gt[0] + res.x;
      gt[1] = gt[1] + res.y;
      gt[2] = gt[2] + res.z;
      const v3 src = vload(ps->inner_surface, nn);
      for (int j = 0; j < 4; ++j) gq[j] = gq[j] + vdot(res, mmul(&dR[j], src));
    }
    mdiv = (double)ncol;
    pt->loss = sum / mdiv;
  } else {
    /* sample_minibatch (spatial_index.cpp:111-131) */
    for (int64_t i = 0; i < P->n_object; ++i) idxbuf[i] = i;
    for (int64_t i = 0; i < m; ++i) {
      const int64_t j = i + (int64_t)uniform_index(rng, (uint64_t)(P->n_object - i));
      const int64_t tmp = idxbuf[i];
      idxbuf[i] = idxbuf[j];
      idxbuf[j] = tmp;
      pool[i] = idxbuf[i];
    }
    /* grasp_gradients + losses (grasp.cpp:37-66) */
    const v3 tcp = {ps->tcp[0], ps->tcp[1], ps->tcp[2]};
    const v3 com = {P->com[0], P->com[1], P->com[2]};
    const v3 cr = vsub(vadd(mmul(&r, tcp), t), com);
    gt[0] = cr.x;
    gt[1] = cr.y;
    gt[2] = cr.z;
    for (int j = 0; j < 4; ++j) gq[j] = vdot(cr, mmul(&dR[j], tcp));
    for (int64_t i = 0; i < ps->n_surface; ++i) {
      const v3 q = vload(sw, i);
      const int64_t nn = nearest(P->object_cloud, pool, m, q);
      const v3 res = vsub(q, vload(P->object_cloud, pool[nn]));
      sum += vsq(res);
      gt[0] = gt[0] + res.x;
      gt[1] = gt[1] + res.y;
      gt[2] = gt[2] + res.z;
      const v3 src = vload(ps->inner_surface, i);
      for (int j = 0; j < 4; ++j) gq[j] = gq[j] + vdot(res, mmul(&dR[j], src));
    }
    mdiv = (double)ps->n_surface;
    pt->loss = sum / mdiv + vsq(cr);
  }
  pt->in_col = ncol > 0;
  for (int a = 0; a < 3; ++a) pt->grad[a] = gt[a] / mdiv;
  for (int a = 0; a < 4; ++a) pt->grad[3 + a] = gq[a] / mdiv;
  /* prior_log_gradient (optim.cpp:146-156) */
  for (int a = 0; a < 3; ++a) {
    const double var = P->prior_t_sigma[a] * P->prior_t_sigma[a];
    pt->prior[a] = -(pt->th[a] - P->prior_t_mean[a]) / var;
  }
  for (int a = 0; a < 4; ++a) pt->prior[3 + a] = -P->prior_q_kappa[a] * sin(pt->th[3 + a] - P->prior_q_location[a]);
}

/* Full-cloud loss for the final ranking (grasp.cpp:263-281). */
static double full_cloud_loss(const asicp_problem* P, const particle* pt, double* sw, int* free_out,
                              int64_t* colbuf) {
  const asicp_preshape* ps = &P->preshapes[pt->pre];
  *free_out = colliding_points(P, &P->sdf_grids[ps->sdf_index], pt->th, colbuf) == 0;
  const m3 r = rotation_matrix(pt->th + 3);
  const v3 t = {pt->th[0], pt->th[1], pt->th[2]};
  double sum = 0.0;
  for (int64_t i = 0; i < ps->n_surface; ++i) {
    const v3 q = vadd(mmul(&r, vload(ps->inner_surface, i)), t);
    const int64_t nn = nearest(P->object_cloud, NULL, P->n_object, q);
    sum += vsq(vsub(q, vload(P->object_cloud, nn)));
  }
  const v3 tcp = {ps->tcp[0], ps->tcp[1], ps->tcp[2]};
  const v3 com = {P->com[0], P->com[1], P->com[2]};
  return sum / (double)ps->n_surface + vsq(vsub(vadd(mmul(&r, tcp), t), com));
  (void)sw;
}

int port_optimize_grasp(const asicp_problem* P, asicp_solution* out, char* err, size_t errlen) {
  if (P->n_object <= 0 || P->n_scene <= 0 || P->n_preshapes <= 0 || P->n_init_lists != P->n_preshapes ||
      P->k_stein > P->k_max) {
    set_err(err, errlen, "invalid problem (see GraspProblem::validate, grasp.cpp:20-31)");
    return ASICP_INVALID_ARGUMENT;
  }
  int64_t J = 0;
  for (int64_t i = 0; i < P->n_init_lists; ++i) J += P->init_counts[i];
  if (J < 1) {
    set_err(err, errlen, "optimize_grasp: no initial poses");
    return ASICP_INVALID_ARGUMENT;
  }
  particle* pts = calloc((size_t)J, sizeof(particle));
  mt64* rngs = malloc((size_t)J * sizeof(mt64));
  int64_t max_ns = 0;
  for (int64_t i = 0; i < P->n_preshapes; ++i)
    if (P->preshapes[i].n_surface > max_ns) max_ns = P->preshapes[i].n_surface;
  int64_t* colbuf = malloc((size_t)P->n_scene * sizeof(int64_t));
  int64_t* idxbuf = malloc((size_t)P->n_object * sizeof(int64_t));
  int64_t* pool = malloc((size_t)P->n_object * sizeof(int64_t));
  double* sw = malloc((size_t)max_ns * 3 * sizeof(double));
  double* dir = malloc((size_t)J * 7 * sizeof(double));
  double* drift = malloc((size_t)J * 7 * sizeof(double));
  int64_t row = 0;
  for (int64_t ps = 0; ps < P->n_preshapes; ++ps)
    for (int64_t k = 0; k < P->init_counts[ps]; ++k, ++row) {
      memcpy(pts[row].th, P->init_poses + 7 * row, 7 * sizeof(double));
      pts[row].pre = (int)ps;
      pts[row].loss = NAN;
      pts[row].prev_loss = NAN;
    }
  for (int64_t j = 0; j < J; ++j) mt_seed(&rngs[j], P->seed + (uint64_t)j); /* grasp.cpp:149-151 */
  const double n_ref = (double)P->n_object;
  const double eta = P->step_scale / n_ref; /* grasp.cpp:154 */
  for (int64_t k = 0; k < P->k_max; ++k) {  /* grasp.cpp:161-258 */
    const int stein = k < P->k_stein;
    const int64_t m = minibatch_schedule(k, P->k_max, P->n_object);
    for (int64_t j = 0; j < J; ++j) {
      if (!stein && pts[j].converged) continue;
      evaluate(P, &pts[j], &rngs[j], m, colbuf, idxbuf, pool, sw);
    }
    if (P->record_trace && out->trace_theta) {
      for (int64_t j = 0; j < J; ++j) {
        memcpy(out->trace_theta + 7 * (k * J + j), pts[j].th, 7 * sizeof(double));
        if (out->trace_loss) out->trace_loss[k * J + j] = pts[j].loss;
        if (out->trace_in_collision) out->trace_in_collision[k * J + j] = pts[j].in_col;
      }
    }
    if (stein) {
      /* annealing (optim.cpp:158-164), svgd_direction / svgd_update (optim.cpp:174-237) */
      const double period = (double)P->anneal_period_total / (double)P->anneal_cycles;
      const double gamma = pow(fmod((double)k, period) / period, P->anneal_exponent);
      int64_t b = 0;
      for (int64_t ps = 0; ps < P->n_preshapes; ++ps) {
        const int64_t K = P->init_counts[ps];
        if (K == 0) continue;
        for (int64_t i = b; i < b + K; ++i)
          for (int a = 0; a < 7; ++a) drift[7 * i + a] = gamma * (n_ref * pts[i].grad[a] + pts[i].prior[a]);
        double h = P->fixed_bandwidth;
        if (P->bandwidth_mode == ASICP_BANDWIDTH_MEDIAN) {
          if (K < 2) {
            h = 1.0;
          } else {
            const int64_t M = K * (K - 1) / 2;
            double* d2 = malloc((size_t)M * sizeof(double));
            int64_t c = 0;
            for (int64_t i = 0; i < K; ++i)
              for (int64_t jj = i + 1; jj < K; ++jj) {
                const v3 ti = {pts[b + i].th[0], pts[b + i].th[1], pts[b + i].th[2]};
                const v3 tj = {pts[b + jj].th[0], pts[b + jj].th[1], pts[b + jj].th[2]};
                d2[c++] = vsq(vsub(ti, tj));
              }
            /* nth_element(d2, M/2): exact order statistic by quickselect */
            int64_t lo = 0, hi = M - 1, want = M / 2;
            while (lo < hi) {
              const double piv = d2[(lo + hi) / 2];
              int64_t i = lo, jj = hi;
              while (i <= jj) {
                while (d2[i] < piv) ++i;
                while (d2[jj] > piv) --jj;
                if (i <= jj) {
                  const double t = d2[i];
                  d2[i] = d2[jj];
                  d2[jj] = t;
                  ++i;
                  --jj;
                }
              }
              if (want <= jj) hi = jj;
              else if (want >= i) lo = i;
              else break;
            }
            const double med = d2[want];
            free(d2);
            h = med / log((double)K + 1.0);
            if (h < 1e-6) h = 1e-6;
          }
        }
        for (int64_t jj = b; jj < b + K; ++jj) {
          double pt_[3] = {0, 0, 0}, pq[4] = {0, 0, 0, 0};
          for (int64_t i = b; i < b + K; ++i) {
            const double* di = drift + 7 * i;
            if (i == jj) {
              for (int a = 0; a < 3; ++a) pt_[a] = pt_[a] - di[a];
              for (int a = 0; a < 4; ++a) pq[a] = pq[a] - di[3 + a];
              continue;
            }
            const v3 ti = {pts[i].th[0], pts[i].th[1], pts[i].th[2]};
            const v3 tj = {pts[jj].th[0], pts[jj].th[1], pts[jj].th[2]};
            const double value = exp(-vsq(vsub(ti, tj)) / h);
            for (int a = 0; a < 3; ++a) pt_[a] = pt_[a] + (-di[a]) * value;
            const double two_h = 2.0 / h;
            const double dt[3] = {tj.x - ti.x, tj.y - ti.y, tj.z - ti.z};
            for (int a = 0; a < 3; ++a) pt_[a] = pt_[a] + (two_h * dt[a]) * value;
            const double dq = ((pts[i].th[3] * pts[jj].th[3] + pts[i].th[4] * pts[jj].th[4]) +
                               pts[i].th[5] * pts[jj].th[5]) + pts[i].th[6] * pts[jj].th[6];
            const double kq = fabs(dq);
            for (int a = 0; a < 4; ++a) pq[a] = pq[a] + (-di[3 + a]) * kq;
          }
          for (int a = 0; a < 3; ++a) dir[7 * jj + a] = pt_[a];
          for (int a = 0; a < 4; ++a) dir[7 * jj + 3 + a] = pq[a];
        }
        for (int64_t jj = b; jj < b + K; ++jj) {
          for (int a = 0; a < 3; ++a) pts[jj].th[a] = pts[jj].th[a] + eta * dir[7 * jj + a];
          for (int a = 0; a < 4; ++a) pts[jj].th[3 + a] = pts[jj].th[3 + a] + eta * dir[7 * jj + 3 + a];
          normalize4(pts[jj].th + 3);
        }
        b += K;
      }
    } else {
      /* sgd_update (optim.cpp:108-114) */
      for (int64_t j = 0; j < J; ++j) {
        if (pts[j].converged) continue;
        double step[7];
        for (int r = 0; r < 7; ++r) {
          double s = P->A[7 * r] * pts[j].grad[0];
          for (int c = 1; c < 7; ++c) s = s + P->A[7 * r + c] * pts[j].grad[c];
          step[r] = P->learning_rate * s;
        }
        for (int a = 0; a < 7; ++a) pts[j].th[a] = pts[j].th[a] - step[a];
        normalize4(pts[j].th + 3);
      }
    }
    /* convergence bookkeeping (grasp.cpp:242-257) */
    for (int64_t j = 0; j < J; ++j) {
      if (stein) {
        pts[j].prev_loss = pts[j].loss;
        continue;
      }
      if (pts[j].converged) continue;
      if (pts[j].in_col) {
        pts[j].converged = 0;
      } else if (isfinite(pts[j].prev_loss) && pts[j].prev_loss > 0.0) {
        pts[j].converged = fabs(pts[j].loss - pts[j].prev_loss) / pts[j].prev_loss <= P->convergence_threshold;
      }
      pts[j].prev_loss = pts[j].loss;
    }
  }
  /* final ranking + selection (grasp.cpp:260-306) */
  int64_t best = -1, attempt = -1;
  double* fl = malloc((size_t)J * sizeof(double));
  int* ff = malloc((size_t)J * sizeof(int));
  for (int64_t j = 0; j < J; ++j) {
    fl[j] = full_cloud_loss(P, &pts[j], sw, &ff[j], colbuf);
    if (ff[j] && (best < 0 || fl[j] < fl[best])) best = j;
    if (attempt < 0 || fl[j] < fl[attempt]) attempt = j;
    if (out->particle_theta) memcpy(out->particle_theta + 7 * j, pts[j].th, 7 * sizeof(double));
    if (out->particle_loss) out->particle_loss[j] = fl[j];
    if (out->particle_collision_free) out->particle_collision_free[j] = ff[j];
    if (out->particle_converged) out->particle_converged[j] = pts[j].converged;
    if (out->particle_preshape) out->particle_preshape[j] = pts[j].pre;
  }
  const int64_t sel = best >= 0 ? best : attempt;
  out->status = best >= 0 ? ASICP_STATUS_FOUND : ASICP_STATUS_NO_GRASP_FOUND;
  memcpy(out->theta, pts[sel].th, 7 * sizeof(double));
  out->preshape_id = pts[sel].pre;
  out->final_loss = fl[sel];
  out->converged = pts[sel].converged;
  out->n_particles = J;
  free(fl);
  free(ff);
  free(pts);
  free(rngs);
  free(colbuf);
  free(idxbuf);
  free(pool);
  free(sw);
  free(dir);
  free(drift);
  return ASICP_OK;
}

/* ------------------------------------------------------------------------
 * graspmatch::register_sgd_icp (optim.cpp:274-321), both preconditioners.
 * ------------------------------------------------------------------------ */

/* SgdConfig::validate (optim.cpp:10-15) via the shim's isApprox / LLT. */
static double a7_norm(const double* A, int transposed) {
  double s = 0.0;
  for (int j = 0; j < 7; ++j)
    for (int i = 0; i < 7; ++i) {
      const double v = transposed ? A[7 * j + i] : A[7 * i + j];
      s = (i == 0 && j == 0) ? v * v : s + v * v;
    }
  return sqrt(s);
}
static const char* sgd_validate(const asicp_sgd_config* c) {
  if (!(c->learning_rate > 0.0)) return "SgdConfig: learning_rate must be positive";
  double d[49], l[7][7];
  for (int i = 0; i < 7; ++i)
    for (int j = 0; j < 7; ++j) d[7 * i + j] = c->A[7 * i + j] - c->A[7 * j + i];
  const double na = a7_norm(c->A, 0), nt = a7_norm(c->A, 1);
  if (!(a7_norm(d, 0) <= 1e-12 * (na < nt ? na : nt))) return "SgdConfig: A must be symmetric";
  for (int i = 0; i < 7; ++i)
    for (int j = 0; j < 7; ++j) l[i][j] = c->A[7 * i + j];
  for (int j = 0; j < 7; ++j) {
    double s = l[j][j];
    for (int k = 0; k < j; ++k) s -= l[j][k] * l[j][k];
    if (!(s > 0.0)) return "SgdConfig: A must be positive definite";
    const double dd = sqrt(s);
    l[j][j] = dd;
    for (int i = j + 1; i < 7; ++i) {
      double t = l[i][j];
      for (int k = 0; k < j; ++k) t -= l[i][k] * l[j][k];
      l[i][j] = t / dd;
    }
    for (int i = 0; i < j; ++i) l[i][j] = 0.0;
  }
  return NULL;
}

/* gauss_newton_rotation_step (optim.cpp:250-270), shim LDLT solve. */
static void gn_step(const double* src, const int64_t* batch, int64_t m, const m3 dR[4], const double* g,
                    double damping, double* dq) {
  double jm[3][4] = {{0}}, mom[4][4] = {{0}}, cen[4][4], a[4][4], l[4][4], dv[4], y[4];
  const double md = (double)m;
  for (int64_t p = 0; p < m; ++p) {
    const v3 s = vload(src, batch[p]);
    v3 v[4];
    for (int j = 0; j < 4; ++j) v[j] = mmul(&dR[j], s);
    for (int j = 0; j < 4; ++j) {
      jm[0][j] = jm[0][j] + v[j].x;
      jm[1][j] = jm[1][j] + v[j].y;
      jm[2][j] = jm[2][j] + v[j].z;
    }
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) mom[i][j] = mom[i][j] + vdot(v[i], v[j]);
  }
  for (int r = 0; r < 3; ++r)
    for (int j = 0; j < 4; ++j) jm[r][j] = jm[r][j] / md;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      cen[i][j] = mom[i][j] / md - ((jm[0][i] * jm[0][j] + jm[1][i] * jm[1][j]) + jm[2][i] * jm[2][j]);
  const double trace = ((cen[0][0] + cen[1][1]) + cen[2][2]) + cen[3][3];
  double gc[4];
  for (int i = 0; i < 4; ++i) gc[i] = g[3 + i] - ((jm[0][i] * g[0] + jm[1][i] * g[1]) + jm[2][i] * g[2]);
  if (!(trace > 1e-12)) {
    for (int i = 0; i < 4; ++i) dq[i] = g[3 + i];
    return;
  }
  const double sd = damping * trace / 4.0;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      a[i][j] = cen[i][j] + sd * (i == j ? 1.0 : 0.0);
      l[i][j] = i == j ? 1.0 : 0.0;
    }
  for (int j = 0; j < 4; ++j) {
    double s = a[j][j];
    for (int k = 0; k < j; ++k) s -= l[j][k] * l[j][k] * dv[k];
    dv[j] = s;
    for (int i = j + 1; i < 4; ++i) {
      double t = a[i][j];
      for (int k = 0; k < j; ++k) t -= l[i][k] * l[j][k] * dv[k];
      l[i][j] = t / dv[j];
    }
  }
  for (int i = 0; i < 4; ++i) {
    double s = gc[i];
    for (int k = 0; k < i; ++k) s -= l[i][k] * y[k];
    y[i] = s;
  }
  for (int i = 0; i < 4; ++i) y[i] /= dv[i];
  for (int i = 3; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < 4; ++k) s -= l[k][i] * dq[k];
    dq[i] = s;
  }
}

int port_register_sgd_icp(const double* src, int64_t ns, const double* ref, int64_t nr, const double* initial,
                          const asicp_sgd_config* c, uint64_t seed, asicp_registration* out, char* err,
                          size_t errlen) {
  if (ns <= 0 || nr <= 0) {
    set_err(err, errlen, "register_sgd_icp: empty cloud");
    return ASICP_INVALID_ARGUMENT;
  }
  const int gn = c->preconditioner_mode == ASICP_PRECOND_GAUSS_NEWTON_ROTATION;
  if (!gn) {
    const char* msg = sgd_validate(c);
    if (msg) {
      set_err(err, errlen, msg);
      return ASICP_INVALID_ARGUMENT;
    }
  }
  mt64* rng = (mt64*)malloc(sizeof(mt64));
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)ns);
  mt_seed(rng, seed);
  const int64_t m = c->minibatch_size < ns ? c->minibatch_size : ns;
  double th[7];
  memcpy(th, initial, sizeof th);
  double prev = -1.0;
  int rc = ASICP_OK;
  out->iterations = 0;
  out->final_loss = 0.0;
  out->converged = 0;
  for (int64_t k = 0; k < c->max_iterations; ++k) {
    /* sample_minibatch_indices (spatial_index.cpp:113-125) */
    if (m < 1) {
      set_err(err, errlen, "sample_minibatch: m out of range");
      rc = ASICP_INVALID_ARGUMENT;
      break;
    }
    for (int64_t i = 0; i < ns; ++i) idx[i] = i;
    for (int64_t i = 0; i < m; ++i) {
      const int64_t j = i + (int64_t)uniform_index(rng, (uint64_t)(ns - i));
      const int64_t v = idx[i];
      idx[i] = idx[j];
      idx[j] = v;
    }
    if (!(fabs(sqrt(qsq(th + 3)) - 1.0) <= 1e-6)) {
      set_err(err, errlen, "rotation_matrix: quaternion is not unit-norm");
      rc = ASICP_INVALID_ARGUMENT;
      break;
    }
    const m3 R = rotation_matrix(th + 3);
    m3 dR[4];
    rotation_derivatives(th + 3, dR);
    const v3 t = {th[0], th[1], th[2]};
    double loss = 0.0, g[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int64_t p = 0; p < m; ++p) {
      const v3 s = vload(src, idx[p]);
      const v3 q = vadd(mmul(&R, s), t);
      const int64_t bi = nearest(ref, NULL, nr, q);
      const v3 rp = vload(ref, bi);
      const double dist = sqrt(vsq(vsub(rp, q)));
      loss = loss + dist * dist;
      const v3 res = vsub(q, rp);
      g[0] = g[0] + res.x;
      g[1] = g[1] + res.y;
      g[2] = g[2] + res.z;
      for (int j = 0; j < 4; ++j) g[3 + j] = g[3 + j] + vdot(res, mmul(&dR[j], s));
    }
    const double md = (double)m;
    loss = loss / md;
    for (int i = 0; i < 7; ++i) g[i] = g[i] / md;
    double pre[7], dq[4];
    for (int r = 0; r < 7; ++r) {
      double s = c->A[7 * r] * g[0];
      for (int k2 = 1; k2 < 7; ++k2) s = s + c->A[7 * r + k2] * g[k2];
      pre[r] = s;
    }
    if (gn)
      gn_step(src, idx, m, dR, g, c->gn_damping, dq);
    else
      for (int i = 0; i < 4; ++i) dq[i] = pre[3 + i];
    for (int i = 0; i < 3; ++i) th[i] = th[i] - c->learning_rate * pre[i];
    for (int i = 0; i < 4; ++i) th[3 + i] = th[3 + i] - c->learning_rate * dq[i];
    normalize4(th + 3);
    out->iterations = k + 1;
    out->final_loss = loss;
    if (prev > 0.0 && c->convergence_threshold >= 0.0 && fabs(loss - prev) / prev <= c->convergence_threshold &&
        m == ns) {
      out->converged = 1;
      break;
    }
    prev = loss;
  }
  memcpy(out->theta, th, sizeof th);
  free(idx);
  free(rng);
  return rc;
}

/* ------------------------------------------------------------------------
 * graspmatch::icp_closed_form_step (optim.cpp:51-90) with the Eigen shim's
 * JacobiSVD (oracle/shim/Eigen/Dense) and quaternion_from_matrix (:29-46).
 * ------------------------------------------------------------------------ */
typedef struct { double a[3][3]; } mat3;

static mat3 mm3(const mat3* x, const mat3* y) {
  mat3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o.a[i][j] = (x->a[i][0] * y->a[0][j] + x->a[i][1] * y->a[1][j]) + x->a[i][2] * y->a[2][j];
  return o;
}
static mat3 tr3(const mat3* x) {
  mat3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o.a[i][j] = x->a[j][i];
  return o;
}
static double det3(const mat3* m) {
  const double(*c)[3] = m->a;
  return (c[0][0] * (c[1][1] * c[2][2] - c[1][2] * c[2][1]) - c[1][0] * (c[0][1] * c[2][2] - c[0][2] * c[2][1])) +
         c[2][0] * (c[0][1] * c[1][2] - c[0][2] * c[1][1]);
}
static double max1(double s) { return 1.0 < s ? s : 1.0; } /* std::max(1.0, s) */

static void svd3(const mat3* in, double sing[3], mat3* U, mat3* V) {
  mat3 u = *in, v = {{{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}};
  for (int sweep = 0; sweep < 100; ++sweep) {
    int rotated = 0;
    for (int p = 0; p < 3; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double alpha = 0, beta = 0, gamma = 0;
        for (int k = 0; k < 3; ++k) {
          alpha += u.a[k][p] * u.a[k][p];
          beta += u.a[k][q] * u.a[k][q];
          gamma += u.a[k][p] * u.a[k][q];
        }
        if (fabs(gamma) <= 1e-300 || fabs(gamma) <= 1e-17 * sqrt(alpha * beta)) continue;
        rotated = 1;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int k = 0; k < 3; ++k) {
          const double up = u.a[k][p], uq = u.a[k][q];
          u.a[k][p] = c * up - s * uq;
          u.a[k][q] = s * up + c * uq;
          const double vp = v.a[k][p], vq = v.a[k][q];
          v.a[k][p] = c * vp - s * vq;
          v.a[k][q] = s * vp + c * vq;
        }
      }
    if (!rotated) break;
  }
  double sv[3];
  for (int j = 0; j < 3; ++j) {
    double s2 = 0.0;
    for (int k = 0; k < 3; ++k) s2 += u.a[k][j] * u.a[k][j];
    sv[j] = sqrt(s2);
  }
  int order[3] = {0, 1, 2}; /* std::sort descending: libstdc++ insertion sort for 3 elements */
  for (int i = 1; i < 3; ++i) {
    const int val = order[i];
    int j = i;
    while (j > 0 && sv[val] > sv[order[j - 1]]) {
      order[j] = order[j - 1];
      --j;
    }
    order[j] = val;
  }
  const double tiny = 1e-300;
  for (int i = 0; i < 3; ++i) {
    const int j = order[i];
    sing[i] = sv[j];
    for (int k = 0; k < 3; ++k) {
      V->a[k][i] = v.a[k][j];
      U->a[k][i] = sv[j] > tiny ? u.a[k][j] / sv[j] : 0.0;
    }
  }
  for (int i = 0; i < 3; ++i) {
    if (sing[i] > tiny * max1(sing[0]) && sing[i] > 0.0) continue;
    for (int trial = 0; trial < 3; ++trial) {
      double cand[3] = {trial == 0 ? 1.0 : 0.0, trial == 1 ? 1.0 : 0.0, trial == 2 ? 1.0 : 0.0};
      for (int k = 0; k < 3; ++k) {
        if (k == i) continue;
        if (k > i && !(sing[k] > 0.0)) continue;
        const double proj = (U->a[0][k] * cand[0] + U->a[1][k] * cand[1]) + U->a[2][k] * cand[2];
        for (int r = 0; r < 3; ++r) cand[r] = cand[r] - U->a[r][k] * proj;
      }
      const double n = sqrt((cand[0] * cand[0] + cand[1] * cand[1]) + cand[2] * cand[2]);
      if (n > 1e-6) {
        for (int r = 0; r < 3; ++r) U->a[r][i] = cand[r] / n;
        break;
      }
    }
  }
}

static void quat_from_matrix(const mat3* m, double* q) {
  const double(*r)[3] = m->a;
  const double tr = (r[0][0] + r[1][1]) + r[2][2];
  if (tr > 0.0) {
    const double s = sqrt(tr + 1.0) * 2.0;
    q[0] = 0.25 * s; q[1] = (r[2][1] - r[1][2]) / s; q[2] = (r[0][2] - r[2][0]) / s; q[3] = (r[1][0] - r[0][1]) / s;
  } else if (r[0][0] > r[1][1] && r[0][0] > r[2][2]) {
    const double s = sqrt(((1.0 + r[0][0]) - r[1][1]) - r[2][2]) * 2.0;
    q[0] = (r[2][1] - r[1][2]) / s; q[1] = 0.25 * s; q[2] = (r[0][1] + r[1][0]) / s; q[3] = (r[0][2] + r[2][0]) / s;
  } else if (r[1][1] > r[2][2]) {
    const double s = sqrt(((1.0 + r[1][1]) - r[0][0]) - r[2][2]) * 2.0;
    q[0] = (r[0][2] - r[2][0]) / s; q[1] = (r[0][1] + r[1][0]) / s; q[2] = 0.25 * s; q[3] = (r[1][2] + r[2][1]) / s;
  } else {
    const double s = sqrt(((1.0 + r[2][2]) - r[0][0]) - r[1][1]) * 2.0;
    q[0] = (r[1][0] - r[0][1]) / s; q[1] = (r[0][2] + r[2][0]) / s; q[2] = (r[1][2] + r[2][1]) / s; q[3] = 0.25 * s;
  }
  normalize4(q);
}

int port_icp_closed_form_step(const double* src, int64_t ns, const double* ref, int64_t nr, const double* theta,
                              asicp_icp_step* out, char* err, size_t errlen) {
  if (ns <= 0 || nr <= 0) {
    set_err(err, errlen, "icp_closed_form_step: empty cloud");
    return ASICP_INVALID_ARGUMENT;
  }
  if (!(fabs(sqrt(qsq(theta + 3)) - 1.0) <= 1e-6)) {
    set_err(err, errlen, "rotation_matrix: quaternion is not unit-norm");
    return ASICP_INVALID_ARGUMENT;
  }
  const m3 R = rotation_matrix(theta + 3);
  const v3 t = {theta[0], theta[1], theta[2]};
  int64_t* match = (int64_t*)malloc(sizeof(int64_t) * (size_t)ns);
  double rm[3] = {0, 0, 0}, sm[3] = {0, 0, 0};
  for (int64_t i = 0; i < ns; ++i) {
    match[i] = nearest(ref, NULL, nr, vadd(mmul(&R, vload(src, i)), t));
    const v3 m = vload(ref, match[i]);
    rm[0] = rm[0] + m.x;
    rm[1] = rm[1] + m.y;
    rm[2] = rm[2] + m.z;
  }
  for (int64_t i = 0; i < ns; ++i)
    for (int a = 0; a < 3; ++a) sm[a] = sm[a] + src[3 * i + a];
  for (int a = 0; a < 3; ++a) {
    sm[a] = sm[a] / (double)ns;
    rm[a] = rm[a] / (double)ns;
  }
  mat3 cov = {{{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}};
  for (int64_t i = 0; i < ns; ++i)
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) cov.a[r][c] = cov.a[r][c] + (src[3 * i + r] - sm[r]) * (ref[3 * match[i] + c] - rm[c]);
  free(match);
  double sing[3];
  mat3 U, V;
  svd3(&cov, sing, &U, &V);
  if (ns < 3 || sing[1] <= 1e-12 * max1(sing[0])) {
    const v3 smv = {sm[0], sm[1], sm[2]};
    const v3 moved = vadd(mmul(&R, smv), t);
    out->theta[0] = theta[0] + (rm[0] - moved.x);
    out->theta[1] = theta[1] + (rm[1] - moved.y);
    out->theta[2] = theta[2] + (rm[2] - moved.z);
    for (int i = 3; i < 7; ++i) out->theta[i] = theta[i];
    out->degenerate = 1;
    return ASICP_OK;
  }
  const mat3 Ut = tr3(&U);
  mat3 D = {{{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}};
  const mat3 VUt = mm3(&V, &Ut);
  D.a[2][2] = det3(&VUt) < 0.0 ? -1.0 : 1.0;
  const mat3 VD = mm3(&V, &D);
  const mat3 r = mm3(&VD, &Ut);
  double q[4];
  quat_from_matrix(&r, q);
  for (int i = 0; i < 3; ++i)
    out->theta[i] = rm[i] - ((r.a[i][0] * sm[0] + r.a[i][1] * sm[1]) + r.a[i][2] * sm[2]);
  for (int i = 0; i < 4; ++i) out->theta[3 + i] = q[i];
  out->degenerate = 0;
  return ASICP_OK;
}
