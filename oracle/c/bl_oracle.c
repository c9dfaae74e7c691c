/*
 * ORACLE -- test infrastructure only.  CPU restatement of the BASELINE-profile
 * refinement path (ESDF build, batched cost/gradient, fixed-step refinement,
 * feasibility flags, best-seed selection).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 *
 * It generalises the reference numba kernels to the 3-D BASELINE shapes:
 *   world hinge^2 cost + in-cell interpolant gradient   planseed/_kernels.py:206-228, :23-57
 *   Jacobian-transpose accumulation along the chain     planseed/_kernels.py:277-289
 *   numpy.gradient smoothness stencils                  planseed/trajopt.py:64-86
 *   row-0 gradient pinned                               planseed/_kernels.py:296-299
 *   analytic box SDF (3-D)                              planseed/_kernels.py:60-83
 *   dense feasibility check (4 interpolants/segment)    planseed/pipeline.py:139-157
 *   select_best tie rules                               planseed/pipeline.py:160-165
 *
 * Arithmetic follows the canonical fp32 operation order written down in DESIGN.md
 * ("Canonical fp32 order"), so the CUDA kernels reproduce it bit for bit.  Build
 * with -ffp-contract=off: every fused multiply-add below is an explicit fmaf().
 * Lane reductions emulate the 32-lane xor butterfly the device uses.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NJ 7
#define LANES 32

static void cs_sincos(float x, float *s, float *c) {
    float j = rintf(x * 0.636619772367581343f);
    int q = (int)j;
    float r = fmaf(-j, 1.5703125f, x);
    r = fmaf(-j, 4.83751296997e-04f, r);
    r = fmaf(-j, 7.54978995489e-08f, r);
    float r2 = r * r;
    float sp = fmaf(fmaf(fmaf(-1.9515295891e-4f, r2, 8.3321608736e-3f), r2, -1.6666654611e-1f) * r2, r, r);
    float cp = fmaf(fmaf(fmaf(fmaf(2.443315711809948e-5f, r2, -1.388731625493765e-3f), r2,
                              4.166664568298827e-2f), r2, -0.5f), r2, 1.0f);
    switch (q & 3) {
        case 0: *s = sp; *c = cp; break;
        case 1: *s = cp; *c = -sp; break;
        case 2: *s = -sp; *c = -cp; break;
        default: *s = -cp; *c = sp; break;
    }
}

static inline void cross3(const float *a, const float *b, float *o) {
    o[0] = fmaf(a[1], b[2], -(a[2] * b[1]));
    o[1] = fmaf(a[2], b[0], -(a[0] * b[2]));
    o[2] = fmaf(a[0], b[1], -(a[1] * b[0]));
}

typedef struct {
    const float *v;
    int nx, ny, nz;
    float ox, oy, oz, inv_h;
} grid_t;

/* trilinear value + in-cell gradient; clamps like planseed/_kernels.py:_bilinear */
static void trilinear(const grid_t *g, const float *p, float *d, float *grad, int *clamped) {
    float ux = (p[0] - g->ox) * g->inv_h;
    float uy = (p[1] - g->oy) * g->inv_h;
    float uz = (p[2] - g->oz) * g->inv_h;
    int cl = (ux < 0.f) | (ux > (float)(g->nx - 1)) | (uy < 0.f) | (uy > (float)(g->ny - 1)) |
             (uz < 0.f) | (uz > (float)(g->nz - 1));
    float fi = fminf(fmaxf(floorf(ux), 0.f), (float)(g->nx - 2));
    float fj = fminf(fmaxf(floorf(uy), 0.f), (float)(g->ny - 2));
    float fk = fminf(fmaxf(floorf(uz), 0.f), (float)(g->nz - 2));
    float tx = fminf(fmaxf(ux - fi, 0.f), 1.f);
    float ty = fminf(fmaxf(uy - fj, 0.f), 1.f);
    float tz = fminf(fmaxf(uz - fk, 0.f), 1.f);
    size_t sy = (size_t)g->nz, sx = (size_t)g->ny * (size_t)g->nz;
    size_t idx = (size_t)(int)fi * sx + (size_t)(int)fj * sy + (size_t)(int)fk;
    const float *v = g->v + idx;
    float v000 = v[0], v001 = v[1], v010 = v[sy], v011 = v[sy + 1];
    float v100 = v[sx], v101 = v[sx + 1], v110 = v[sx + sy], v111 = v[sx + sy + 1];
    float z00 = v001 - v000, z01 = v011 - v010, z10 = v101 - v100, z11 = v111 - v110;
    float c00 = fmaf(tz, z00, v000), c01 = fmaf(tz, z01, v010);
    float c10 = fmaf(tz, z10, v100), c11 = fmaf(tz, z11, v110);
    float e0 = c01 - c00, e1 = c11 - c10;
    float c0 = fmaf(ty, e0, c00), c1 = fmaf(ty, e1, c10);
    float dxv = c1 - c0;
    *d = fmaf(tx, dxv, c0);
    float dyv = fmaf(tx, e1 - e0, e0);
    float zy0 = fmaf(ty, z01 - z00, z00), zy1 = fmaf(ty, z11 - z10, z10);
    float dzv = fmaf(tx, zy1 - zy0, zy0);
    grad[0] = dxv * g->inv_h;
    grad[1] = dyv * g->inv_h;
    grad[2] = dzv * g->inv_h;
    *clamped = cl;
}

typedef struct {
    const float *dh;       /* (7,4): a, d, cos alpha, sin alpha */
    const float *base;     /* (3,) */
    const float *sph;      /* (S,4): x, y, z, r in link frame */
    const int *sph_link;   /* (S,) sorted */
    int n_sph;
} robot_t;

typedef struct {
    float w_coll, w_vel, w_acc, w_jerk, margin, eta;
} cost_t;

/* One configuration: world cost, joint gradient of the world cost, min clearance
 * (d - r) and clamped flag.  want_grad=0 skips the gradient. */
static void config_world(const robot_t *rb, const grid_t *g, const cost_t *w, const float *q,
                         int want_grad, float *cost_out, float *gq, float *minclear, int *clamped) {
    float X[3] = {1.f, 0.f, 0.f}, Y[3] = {0.f, 1.f, 0.f}, Z[3] = {0.f, 0.f, 1.f};
    float o[3] = {rb->base[0], rb->base[1], rb->base[2]};
    float tz[NJ][3], tm[NJ][3];
    float wc = 0.f, mc = INFINITY;
    int cl_any = 0;
    float m2w = -2.0f * w->w_coll;
    int s = 0;
    for (int j = 0; j < NJ; ++j) gq[j] = 0.f;
    for (int k = 0; k < NJ; ++k) {
        tz[k][0] = Z[0]; tz[k][1] = Z[1]; tz[k][2] = Z[2];
        cross3(o, Z, tm[k]);
        float sn, cs;
        cs_sincos(q[k], &sn, &cs);
        const float a = rb->dh[4 * k], dd = rb->dh[4 * k + 1], ca = rb->dh[4 * k + 2], sa = rb->dh[4 * k + 3];
        float ac = a * cs, as = a * sn;
        for (int i = 0; i < 3; ++i) o[i] = fmaf(ac, X[i], fmaf(as, Y[i], fmaf(dd, Z[i], o[i])));
        float X1[3], Y1[3], Y2[3], Z2[3];
        for (int i = 0; i < 3; ++i) {
            X1[i] = fmaf(cs, X[i], sn * Y[i]);
            Y1[i] = fmaf(cs, Y[i], -(sn * X[i]));
        }
        for (int i = 0; i < 3; ++i) {
            Y2[i] = fmaf(ca, Y1[i], sa * Z[i]);
            Z2[i] = fmaf(ca, Z[i], -(sa * Y1[i]));
        }
        for (int i = 0; i < 3; ++i) { X[i] = X1[i]; Y[i] = Y2[i]; Z[i] = Z2[i]; }
        float S1[3] = {0.f, 0.f, 0.f}, S2[3] = {0.f, 0.f, 0.f};
        for (; s < rb->n_sph && rb->sph_link[s] == k; ++s) {
            const float *sp = rb->sph + 4 * s;
            float p[3];
            for (int i = 0; i < 3; ++i) p[i] = fmaf(X[i], sp[0], fmaf(Y[i], sp[1], fmaf(Z[i], sp[2], o[i])));
            float dv, gr[3];
            int cl;
            trilinear(g, p, &dv, gr, &cl);
            cl_any |= cl;
            float clr = dv - sp[3];
            mc = fminf(mc, clr);
            float hinge = (sp[3] + w->margin) - dv;
            if (hinge > 0.f) {
                wc = fmaf(w->w_coll * hinge, hinge, wc);
                if (want_grad) {
                    float coef = m2w * hinge;
                    float gp[3] = {coef * gr[0], coef * gr[1], coef * gr[2]};
                    float cr[3];
                    cross3(p, gp, cr);
                    for (int i = 0; i < 3; ++i) { S1[i] = S1[i] + cr[i]; S2[i] = S2[i] + gp[i]; }
                }
            }
        }
        if (want_grad) {
            for (int j = 0; j <= k; ++j) {
                float t = tz[j][0] * S1[0];
                t = fmaf(tz[j][1], S1[1], t);
                t = fmaf(tz[j][2], S1[2], t);
                t = fmaf(tm[j][0], S2[0], t);
                t = fmaf(tm[j][1], S2[1], t);
                t = fmaf(tm[j][2], S2[2], t);
                gq[j] = gq[j] + t;
            }
        }
    }
    *cost_out = wc;
    *minclear = mc;
    *clamped = cl_any;
}

/* 3-term stencils of D (numpy.gradient) and D^T at waypoint t of T */
static inline float stencil(const float *y, int t, int T, int transpose) {
    float cl, cs, cr;
    if (!transpose) {
        cs = (t == 0) ? -1.f : (t == T - 1 ? 1.f : 0.f);
        cl = (t == 0) ? 0.f : (t == T - 1 ? -1.f : -0.5f);
        cr = (t == T - 1) ? 0.f : (t == 0 ? 1.f : 0.5f);
    } else {
        cs = (t == 0) ? -1.f : (t == T - 1 ? 1.f : 0.f);
        cl = (t == 0) ? 0.f : (t - 1 == 0 ? 1.f : 0.5f);
        cr = (t == T - 1) ? 0.f : (t + 1 == T - 1 ? -1.f : -0.5f);
    }
    float ym = y[t > 0 ? t - 1 : t], yp = y[t < T - 1 ? t + 1 : t];
    float r = cs * y[t];
    r = fmaf(cl, ym, r);
    r = fmaf(cr, yp, r);
    return r;
}

/* smoothness cost per waypoint (sm[t]) and gradient (gs[t][k]) of one trajectory */
static void smooth_terms(const float *q, int T, const cost_t *w, float *sm, float *gs) {
    float y[128], v[128], a[128], jk[128], z[128], zz[128];
    for (int t = 0; t < T; ++t) sm[t] = 0.f;
    for (int k = 0; k < NJ; ++k) {
        for (int t = 0; t < T; ++t) y[t] = q[t * NJ + k];
        for (int t = 0; t < T; ++t) v[t] = stencil(y, t, T, 0);
        for (int t = 0; t < T; ++t) a[t] = stencil(v, t, T, 0);
        for (int t = 0; t < T; ++t) jk[t] = stencil(a, t, T, 0);
        for (int t = 0; t < T; ++t) {
            float s = sm[t];
            s = fmaf(w->w_vel, v[t] * v[t], s);
            s = fmaf(w->w_acc, a[t] * a[t], s);
            s = fmaf(w->w_jerk, jk[t] * jk[t], s);
            sm[t] = s;
        }
        if (gs) {
            for (int t = 0; t < T; ++t) z[t] = w->w_jerk * jk[t];
            for (int t = 0; t < T; ++t) zz[t] = fmaf(w->w_acc, a[t], stencil(z, t, T, 1));
            for (int t = 0; t < T; ++t) z[t] = fmaf(w->w_vel, v[t], stencil(zz, t, T, 1));
            for (int t = 0; t < T; ++t) gs[t * NJ + k] = stencil(z, t, T, 1);
        }
    }
}

/* emulate the device's xor butterfly over 32 lanes; lane l holds waypoints l*wpl.. */
static float lane_sum(const float *per_t, int T) {
    int wpl = T / LANES;
    float lanes[LANES];
    for (int l = 0; l < LANES; ++l) {
        float s = per_t[l * wpl];
        for (int i = 1; i < wpl; ++i) s = s + per_t[l * wpl + i];
        lanes[l] = s;
    }
    for (int off = 16; off >= 1; off >>= 1) {
        float nw[LANES];
        for (int l = 0; l < LANES; ++l) nw[l] = lanes[l] + lanes[l ^ off];
        memcpy(lanes, nw, sizeof(lanes));
    }
    return lanes[0];
}

static void setup(grid_t *g, const float *esdf, const int *n, const float *origin, float h) {
    g->v = esdf;
    g->nx = n[0]; g->ny = n[1]; g->nz = n[2];
    g->ox = origin[0]; g->oy = origin[1]; g->oz = origin[2];
    g->inv_h = 1.0f / h;
}

/* ------------------------------------------------------------------------- */

/* analytic box SDF on the grid nodes; node (i,j,k) at origin + h*(i,j,k) */
void orc_esdf_build(const float *boxes, int n_boxes, const int *n, const float *origin, float h,
                    float cap, float *out) {
    for (int i = 0; i < n[0]; ++i)
        for (int j = 0; j < n[1]; ++j)
            for (int k = 0; k < n[2]; ++k) {
                float p[3] = {fmaf((float)i, h, origin[0]), fmaf((float)j, h, origin[1]),
                              fmaf((float)k, h, origin[2])};
                float best = cap;
                for (int b = 0; b < n_boxes; ++b) {
                    const float *bx = boxes + 6 * b;
                    float qd[3];
                    for (int a = 0; a < 3; ++a) {
                        float c = 0.5f * (bx[a] + bx[3 + a]);
                        float hw = 0.5f * (bx[3 + a] - bx[a]);
                        qd[a] = fabsf(p[a] - c) - hw;
                    }
                    float ax = fmaxf(qd[0], 0.f), ay = fmaxf(qd[1], 0.f), az = fmaxf(qd[2], 0.f);
                    float outside = sqrtf(fmaf(ax, ax, fmaf(ay, ay, az * az)));
                    float inside = fminf(fmaxf(qd[0], fmaxf(qd[1], qd[2])), 0.f);
                    float dd = outside + inside;
                    best = fminf(best, dd);
                }
                out[((size_t)i * n[1] + j) * n[2] + k] = best;
            }
}

/* cost (S,) and gradient (S,T,7) of B trajectories; traj b uses problem b / S */
void orc_bl_cost(const float *q, int B, int T, int S, const float *esdf, long long esdf_stride,
                 const int *n, const float *origin, float h, const float *dh, const float *base,
                 const float *sph, const int *sph_link, int n_sph, const float *wts, float *cost,
                 float *grad, int *clamped) {
    robot_t rb = {dh, base, sph, sph_link, n_sph};
    cost_t w = {wts[0], wts[1], wts[2], wts[3], wts[4], wts[5]};
    float *sm = (float *)malloc(sizeof(float) * T);
    float *gs = (float *)malloc(sizeof(float) * T * NJ);
    float *ct = (float *)malloc(sizeof(float) * T);
    for (int b = 0; b < B; ++b) {
        grid_t g;
        setup(&g, esdf + (size_t)(b / S) * (size_t)esdf_stride, n, origin, h);
        const float *qb = q + (size_t)b * T * NJ;
        smooth_terms(qb, T, &w, sm, gs);
        int cl_any = 0;
        for (int t = 0; t < T; ++t) {
            float wc, mc, gq[NJ];
            int cl;
            config_world(&rb, &g, &w, qb + t * NJ, 1, &wc, gq, &mc, &cl);
            cl_any |= cl;
            ct[t] = wc + sm[t];
            for (int k = 0; k < NJ; ++k) {
                float gg = fmaf(2.0f, gs[t * NJ + k], gq[k]);
                grad[((size_t)b * T + t) * NJ + k] = (t == 0) ? 0.f : gg;
            }
        }
        cost[b] = lane_sum(ct, T);
        if (clamped) clamped[b] = cl_any;
    }
    free(sm); free(gs); free(ct);
}

/* n_iters fixed steps, then final cost, feasibility and clamped flags */
void orc_bl_refine(const float *q_in, int B, int T, int S, const float *esdf, long long esdf_stride,
                   const int *n, const float *origin, float h, const float *dh, const float *base,
                   const float *sph, const int *sph_link, int n_sph, const float *wts, int n_iters,
                   float *q_out, float *cost, int *feasible, int *clamped) {
    robot_t rb = {dh, base, sph, sph_link, n_sph};
    cost_t w = {wts[0], wts[1], wts[2], wts[3], wts[4], wts[5]};
    float *sm = (float *)malloc(sizeof(float) * T);
    float *gs = (float *)malloc(sizeof(float) * T * NJ);
    float *ct = (float *)malloc(sizeof(float) * T);
    float *x = (float *)malloc(sizeof(float) * T * NJ);
    for (int b = 0; b < B; ++b) {
        grid_t g;
        setup(&g, esdf + (size_t)(b / S) * (size_t)esdf_stride, n, origin, h);
        memcpy(x, q_in + (size_t)b * T * NJ, sizeof(float) * T * NJ);
        for (int it = 0; it < n_iters; ++it) {
            float gw[128][NJ];
            for (int t = 0; t < T; ++t) {
                float wc, mc;
                int cl;
                config_world(&rb, &g, &w, x + t * NJ, 1, &wc, gw[t], &mc, &cl);
            }
            smooth_terms(x, T, &w, sm, gs);
            for (int t = 1; t < T; ++t)
                for (int k = 0; k < NJ; ++k) {
                    float gg = fmaf(2.0f, gs[t * NJ + k], gw[t][k]);
                    x[t * NJ + k] = fmaf(-w.eta, gg, x[t * NJ + k]);
                }
        }
        smooth_terms(x, T, &w, sm, NULL);
        float mc_all = INFINITY;
        int cl_any = 0;
        for (int t = 0; t < T; ++t) {
            float wc, mc, gq[NJ];
            int cl;
            config_world(&rb, &g, &w, x + t * NJ, 0, &wc, gq, &mc, &cl);
            ct[t] = wc + sm[t];
            mc_all = fminf(mc_all, mc);
            cl_any |= cl;
        }
        for (int t = 0; t + 1 < T; ++t)
            for (int i = 0; i < 4; ++i) {
                float f = (float)(i + 1) / 5.0f;
                float qi[NJ], wc, mc, gq[NJ];
                int cl;
                for (int k = 0; k < NJ; ++k)
                    qi[k] = fmaf(f, x[(t + 1) * NJ + k] - x[t * NJ + k], x[t * NJ + k]);
                config_world(&rb, &g, &w, qi, 0, &wc, gq, &mc, &cl);
                mc_all = fminf(mc_all, mc);
                cl_any |= cl;
            }
        cost[b] = lane_sum(ct, T);
        feasible[b] = mc_all > 0.f;   /* clamped lookups count with clamped values, as planner_success */
        clamped[b] = cl_any;
        memcpy(q_out + (size_t)b * T * NJ, x, sizeof(float) * T * NJ);
    }
    free(sm); free(gs); free(ct); free(x);
}

/* one trajectory's cost (and gradient, row 0 zero, when grad != NULL); as orc_bl_cost */
static float traj_cost(const robot_t *rb, const grid_t *g, const cost_t *w, const float *q, int T, float *grad,
                       int *clamped, float *sm, float *gs, float *ct) {
    smooth_terms(q, T, w, sm, grad ? gs : NULL);
    int cl_any = 0;
    for (int t = 0; t < T; ++t) {
        float wc, mc, gq[NJ];
        int cl;
        config_world(rb, g, w, q + t * NJ, grad ? 1 : 0, &wc, gq, &mc, &cl);
        cl_any |= cl;
        ct[t] = wc + sm[t];
        if (grad)
            for (int k = 0; k < NJ; ++k) grad[t * NJ + k] = (t == 0) ? 0.f : fmaf(2.0f, gs[t * NJ + k], gq[k]);
    }
    *clamped = cl_any;
    return lane_sum(ct, T);
}

/* guided_ddim_sample's guide() (planseed/diffusion.py:598-617) for the BL cost on normalised
 * x0_hat (B,T,7), in place: n_grad descent steps, each from step alpha with <= max_halvings
 * halvings until the cost of the denormalised candidate (lo + x * span) decreases.
 * clamped[b] = some evaluation of trajectory b left the ESDF extent. */
void orc_bl_guide(float *x, int B, int T, int S, const float *esdf, long long esdf_stride, const int *n,
                  const float *origin, float h, const float *dh, const float *base, const float *sph,
                  const int *sph_link, int n_sph, const float *wts, const float *lo, const float *span,
                  int n_grad, float alpha, int max_halvings, int *clamped) {
    robot_t rb = {dh, base, sph, sph_link, n_sph};
    cost_t w = {wts[0], wts[1], wts[2], wts[3], wts[4], wts[5]};
    float *sm = (float *)malloc(sizeof(float) * T), *gs = (float *)malloc(sizeof(float) * T * NJ);
    float *ct = (float *)malloc(sizeof(float) * T), *q = (float *)malloc(sizeof(float) * T * NJ);
    float *gr = (float *)malloc(sizeof(float) * T * NJ), *cand = (float *)malloc(sizeof(float) * T * NJ);
    for (int b = 0; b < B; ++b) {
        grid_t g;
        setup(&g, esdf + (size_t)(b / S) * (size_t)esdf_stride, n, origin, h);
        float *xb = x + (size_t)b * T * NJ;
        int cl_any = 0, cl;
        for (int it = 0; it < n_grad; ++it) {
            for (int i = 0; i < T * NJ; ++i) q[i] = lo[i % NJ] + xb[i] * span[i % NJ];
            const float c = traj_cost(&rb, &g, &w, q, T, gr, &cl, sm, gs, ct);
            cl_any |= cl;
            for (int i = 0; i < T * NJ; ++i) gr[i] = gr[i] * span[i % NJ];
            float step = alpha;
            for (int hv = 0; hv < max_halvings; ++hv) {
                for (int i = 0; i < T * NJ; ++i) {
                    cand[i] = xb[i] - step * gr[i];
                    q[i] = lo[i % NJ] + cand[i] * span[i % NJ];
                }
                const float cn = traj_cost(&rb, &g, &w, q, T, NULL, &cl, sm, gs, ct);
                cl_any |= cl;
                if (cn < c) {
                    memcpy(xb, cand, sizeof(float) * T * NJ);
                    break;
                }
                step = step * 0.5f;
            }
        }
        clamped[b] = cl_any;
    }
    free(sm); free(gs); free(ct); free(q); free(gr); free(cand);
}

/* lowest-cost feasible seed, else lowest cost; ties to the lower index */
void orc_select(const float *cost, const int *feasible, int P, int S, int *best) {
    for (int p = 0; p < P; ++p) {
        int any = 0;
        for (int s = 0; s < S; ++s) any |= feasible[p * S + s];
        int bi = -1;
        float bc = 0.f;
        for (int s = 0; s < S; ++s) {
            if (any && !feasible[p * S + s]) continue;
            float c = cost[p * S + s];
            if (bi < 0 || c < bc) { bi = s; bc = c; }
        }
        best[p] = bi;
    }
}

/* Philox4x32-10 (Salmon et al., SC'11) */
void orc_philox(const uint32_t *ctr_in, const uint32_t *key_in, uint32_t *out) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}
