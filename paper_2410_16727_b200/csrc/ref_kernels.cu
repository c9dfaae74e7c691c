// Reference-profile ("ref") kernels: planseed's own planar arm, 5-term cost, momentum +
// Armijo optimiser, FC denoiser, scan encoder, scan-derived ESDF and planner_success,
// on the GPU behind the numba/numpy signatures.  Templated on the scalar type: the
// double instantiation is the parity mode against planseed itself (compiled with
// --fmad=false and the reference's evaluation order, so results agree to ~1e-13), the
// float instantiation the fast mode.
//
// Reference: src/_kernels.py:18-57 (_wrap, _bilinear), :165-312 (cost_terms_batch),
// :315-431 (optimize_batch); src/diffusion.py:207-300 (features, encoder, denoiser);
// src/pipeline.py:101-157 (planner ESDF, planner_success).
#include <cuda_bf16.h>

#include <cooperative_groups.h>

#include <cmath>

#include "common.cuh"

namespace ps {
namespace ref {

constexpr int MAXD = 8;        // joints
constexpr int MAXM = 8;        // points per link
constexpr int MAXP = MAXD * MAXM;
constexpr int MAXPAIR = 512;
constexpr int MAXT = 64;       // waypoints

template <typename F>
struct ArmGrid {
    int D, M, n_pairs;
    F lengths[MAXD];
    F fracs[MAXM];
    F basex, basey;
    short pair_a[MAXPAIR], pair_b[MAXPAIR];
    const F* grid;
    int nx, ny;
    F gox, goy, gh;
    F goal_x, goal_y, goal_th;
    F w[5];
    F d_act, d_self;
    const F* jerk_mat;   // (T,T)
    const F* jerk_quad;  // (T,T)
};

// Python float modulo (CPython float_rem): sign follows the divisor.
template <typename F>
__device__ __forceinline__ F py_mod(F a, F b) {
    F m = fmod(a, b);
    if (m != F(0)) {
        if ((b < F(0)) != (m < F(0))) m += b;
    } else {
        m = copysign(F(0), b);
    }
    return m;
}

template <typename F>
__device__ __forceinline__ F wrap(F th) {
    const F pi = F(3.141592653589793238462643383279502884);
    return pi - py_mod(pi - th, F(2) * pi);
}

template <typename F>
__device__ __forceinline__ F floorT(F x) { return floor(x); }

// _bilinear (src/_kernels.py:23-57), same expression order
template <typename F>
__device__ void bilinear(const ArmGrid<F>& A, F x, F y, F& d, F& dgx, F& dgy, bool& clamped) {
    const int nx = A.nx, ny = A.ny;
    const F gx = (x - A.gox) / A.gh;
    const F gy = (y - A.goy) / A.gh;
    clamped = gx < F(0) || gx > F(nx - 1) || gy < F(0) || gy > F(ny - 1);
    // int(np.floor(gx)) then clamp; guard the conversion for far-out points
    F fx = floorT(gx), fy = floorT(gy);
    int i = fx < F(0) ? -1 : (fx > F(nx) ? nx : (int)fx);
    int j = fy < F(0) ? -1 : (fy > F(ny) ? ny : (int)fy);
    if (i < 0) i = 0; else if (i > nx - 2) i = nx - 2;
    if (j < 0) j = 0; else if (j > ny - 2) j = ny - 2;
    F tx = gx - F(i), ty = gy - F(j);
    if (tx < F(0)) tx = F(0); else if (tx > F(1)) tx = F(1);
    if (ty < F(0)) ty = F(0); else if (ty > F(1)) ty = F(1);
    const F* v = A.grid;
    const F v00 = v[(size_t)i * ny + j], v10 = v[(size_t)(i + 1) * ny + j];
    const F v01 = v[(size_t)i * ny + j + 1], v11 = v[(size_t)(i + 1) * ny + j + 1];
    d = v00 * (1 - tx) * (1 - ty) + v10 * tx * (1 - ty) + v01 * (1 - tx) * ty + v11 * tx * ty;
    dgx = ((v10 - v00) * (1 - ty) + (v11 - v01) * ty) / A.gh;
    dgy = ((v01 - v00) * (1 - tx) + (v11 - v10) * tx) / A.gh;
}

// Per-warp scratch in shared memory for one seed.
template <typename F>
struct SeedScratch {
    F world[MAXT][MAXP];   // per (t, p) world-term contributions (0 when inactive)
    F self_[MAXT];
    F smooth[MAXD][MAXT];
    F goal_pos, goal_rot;
    int clamped;
};

// One waypoint (lane-owned): world + self + goal terms and the joint gradient
// (goal-rot part, then the backward accumulation), as cost_terms_batch does.
template <typename F>
__device__ void waypoint_terms(const ArmGrid<F>& A, const F* q, int t, int T, bool want_grad,
                               SeedScratch<F>& sc, F* gq) {
    const int D = A.D, M = A.M, P = D * M;
    F ox[MAXD + 1], oy[MAXD + 1], px[MAXP], py[MAXP], gpx[MAXP], gpy[MAXP], cth[MAXD];
    F th = 0;
    ox[0] = A.basex;
    oy[0] = A.basey;
    for (int k = 0; k < D; ++k) {
        th += q[k];
        cth[k] = th;
        const F c = cos(th), si = sin(th);
        for (int i = 0; i < M; ++i) {
            const int p = k * M + i;
            px[p] = ox[k] + A.fracs[i] * A.lengths[k] * c;
            py[p] = oy[k] + A.fracs[i] * A.lengths[k] * si;
        }
        ox[k + 1] = ox[k] + A.lengths[k] * c;
        oy[k + 1] = oy[k] + A.lengths[k] * si;
    }
    for (int p = 0; p < P; ++p) gpx[p] = gpy[p] = 0;
    bool any_point_grad = false;
    const F w_gp = A.w[0], w_gr = A.w[1], w_self = A.w[3], w_world = A.w[4];
    for (int p = 0; p < P; ++p) sc.world[t][p] = 0;
    if (w_world > F(0)) {
        for (int p = 0; p < P; ++p) {
            F dv, dgx, dgy;
            bool cl;
            bilinear(A, px[p], py[p], dv, dgx, dgy, cl);
            if (cl) sc.clamped = 1;
            const F hinge = A.d_act - dv;
            if (hinge > F(0)) {
                sc.world[t][p] = w_world * hinge * hinge;
                if (want_grad) {
                    gpx[p] += F(-2.0) * w_world * hinge * dgx;
                    gpy[p] += F(-2.0) * w_world * hinge * dgy;
                    any_point_grad = true;
                }
            }
        }
    }
    sc.self_[t] = 0;
    if (w_self > F(0) && A.n_pairs > 0) {
        F best = F(1e300 > 3e38 && sizeof(F) == 4 ? 3.0e38 : 1e300);
        int best_i = 0;
        for (int e = 0; e < A.n_pairs; ++e) {
            const int a = A.pair_a[e], b = A.pair_b[e];
            const F dx = px[a] - px[b], dy = py[a] - py[b];
            const F dd = dx * dx + dy * dy;
            if (dd < best) {
                best = dd;
                best_i = e;
            }
        }
        const F mind = sqrt(best);
        const F hinge = A.d_self - mind;
        if (hinge > F(0)) {
            sc.self_[t] = w_self * hinge * hinge;
            if (want_grad && mind > F(1e-12)) {
                const int a = A.pair_a[best_i], b = A.pair_b[best_i];
                const F scale = F(-2.0) * w_self * hinge / mind;
                gpx[a] += scale * (px[a] - px[b]);
                gpy[a] += scale * (py[a] - py[b]);
                gpx[b] += -scale * (px[a] - px[b]);
                gpy[b] += -scale * (py[a] - py[b]);
                any_point_grad = true;
            }
        }
    }
    for (int k = 0; k < D; ++k) gq[k] = 0;
    F ee_gx = 0, ee_gy = 0;
    if (t == T - 1) {
        const F ex = ox[D] - A.goal_x, ey = oy[D] - A.goal_y;
        sc.goal_pos = w_gp * (ex * ex + ey * ey);
        const F dth = wrap(cth[D - 1] - A.goal_th);
        sc.goal_rot = w_gr * dth * dth;
        if (want_grad) {
            ee_gx = F(2.0) * w_gp * ex;
            ee_gy = F(2.0) * w_gp * ey;
            for (int k = 0; k < D; ++k) gq[k] += F(2.0) * w_gr * dth;
        }
    }
    if (want_grad && (any_point_grad || ee_gx != F(0) || ee_gy != F(0))) {
        F acc = ee_gy * ox[D] - ee_gx * oy[D];
        F bx = ee_gx, by = ee_gy;
        for (int k = D - 1; k >= 0; --k) {
            for (int i = 0; i < M; ++i) {
                const int p = k * M + i;
                acc += gpy[p] * px[p] - gpx[p] * py[p];
                bx += gpx[p];
                by += gpy[p];
            }
            gq[k] += acc - ox[k] * by + oy[k] * bx;
        }
    }
}

// Full cost of one seed by one warp.  q: smem (T, D).  grad (optional): smem (T, D).
// Returns total (all lanes), writes terms[5] (lane 0) and clamped.
template <typename F>
__device__ F seed_cost(const ArmGrid<F>& A, const F* q, int T, bool want_grad, SeedScratch<F>& sc, F* grad,
                       F* terms, int& clamped) {
    const int lane = threadIdx.x & 31;
    const int D = A.D, P = A.D * A.M;
    if (lane == 0) {
        sc.clamped = 0;
        sc.goal_pos = sc.goal_rot = 0;
    }
    __syncwarp();
    for (int t = lane; t < T; t += 32) {
        F gq[MAXD];
        waypoint_terms(A, q + t * D, t, T, want_grad, sc, gq);
        if (want_grad)
            for (int k = 0; k < D; ++k) grad[t * D + k] = gq[k];
    }
    __syncwarp();
    // smoothness: y = J q per (k, r); gradient w_sm * (2 J^T J q)
    const F w_sm = A.w[2];
    if (w_sm > F(0)) {
        for (int idx = lane; idx < D * T; idx += 32) {
            const int k = idx / T, r = idx % T;
            F y = 0;
            for (int c = 0; c < T; ++c) y += A.jerk_mat[r * T + c] * q[c * D + k];
            sc.smooth[k][r] = w_sm * y * y;
        }
        __syncwarp();
        if (want_grad) {
            for (int idx = lane; idx < D * T; idx += 32) {
                const int k = idx / T, r = idx % T;
                F g = 0;
                for (int c = 0; c < T; ++c) g += A.jerk_quad[r * T + c] * q[c * D + k];
                grad[r * D + k] += w_sm * g;
            }
        }
    }
    __syncwarp();
    F total = 0;
    if (lane == 0) {
        F tw = 0, ts = 0, tsm = 0;
        for (int t = 0; t < T; ++t)
            for (int p = 0; p < P; ++p) tw += sc.world[t][p];
        for (int t = 0; t < T; ++t) ts += sc.self_[t];
        if (w_sm > F(0))
            for (int k = 0; k < D; ++k)
                for (int r = 0; r < T; ++r) tsm += sc.smooth[k][r];
        terms[0] = sc.goal_pos;
        terms[1] = sc.goal_rot;
        terms[2] = tsm;
        terms[3] = ts;
        terms[4] = tw;
        total = terms[0] + terms[1] + terms[2] + terms[3] + terms[4];
    }
    if (want_grad)
        for (int k = lane; k < D; k += 32) grad[k] = 0;  // row 0 pinned
    __syncwarp();
    clamped = sc.clamped;
    return __shfl_sync(PS_FULL, total, 0);
}

template <typename F>
struct SeedSmem {
    SeedScratch<F> sc;
    F q[MAXT * MAXD];
    F g[MAXT * MAXD];
    F v[MAXT * MAXD];
    F cand[MAXT * MAXD];
    F terms[5];
};

template <typename F>
__global__ void __launch_bounds__(32) cost_kernel(const __grid_constant__ ArmGrid<F> A, const F* __restrict__ qs, int S,
                                                  int T, int want_grad, F* terms_out, F* totals, F* grads,
                                                  uint8_t* clamped) {
    extern __shared__ __align__(16) uint8_t smraw[];
    SeedSmem<F>& sm = *reinterpret_cast<SeedSmem<F>*>(smraw);
    const int s = blockIdx.x, lane = threadIdx.x;
    const int n = T * A.D;
    for (int i = lane; i < n; i += 32) sm.q[i] = qs[(size_t)s * n + i];
    __syncwarp();
    int cl;
    const F tot = seed_cost(A, sm.q, T, want_grad != 0, sm.sc, sm.g, sm.terms, cl);
    __syncwarp();
    if (lane == 0) {
        for (int i = 0; i < 5; ++i) terms_out[s * 5 + i] = sm.terms[i];
        totals[s] = tot;
        clamped[s] = (uint8_t)(cl ? 1 : 0);
    }
    for (int i = lane; i < n; i += 32) grads[(size_t)s * n + i] = want_grad ? sm.g[i] : F(0);
}

// optimize_batch (src/_kernels.py:315-431): one warp per seed, identical control flow.
template <typename F>
__global__ void __launch_bounds__(32) optimize_kernel(const __grid_constant__ ArmGrid<F> A, const F* __restrict__ seeds,
                                                      int S, int T, int n_iters, F momentum, F armijo_c, F shrink,
                                                      int max_backtracks, F alpha0, F alpha_max, F* x_out,
                                                      F* terms_out, F* totals, uint8_t* frozen_out,
                                                      long long* n_acc_out) {
    extern __shared__ __align__(16) uint8_t smraw[];
    SeedSmem<F>& sm = *reinterpret_cast<SeedSmem<F>*>(smraw);
    const int s = blockIdx.x, lane = threadIdx.x;
    const int n = T * A.D;
    for (int i = lane; i < n; i += 32) {
        sm.q[i] = seeds[(size_t)s * n + i];
        sm.v[i] = 0;
    }
    __syncwarp();
    F alpha = alpha0;
    bool frozen = false;
    long long n_acc = 0;
    int cl;
    F f = seed_cost(A, sm.q, T, true, sm.sc, sm.g, sm.terms, cl);
    const F INF = F(INFINITY);
    for (int it = 0; it < n_iters; ++it) {
        if (frozen) break;  // a frozen seed never changes again (the batch loop skips it)
        if (it > 0) {
            F dummy_terms[5];
            (void)dummy_terms;
            seed_cost(A, sm.q, T, true, sm.sc, sm.g, sm.terms, cl);
        }
        __syncwarp();
        // gmax and vzero (order-independent)
        F gmax = 0;
        bool vzero = true;
        for (int i = lane; i < n; i += 32) {
            const F ag = fabs(sm.g[i]);
            if (ag > gmax) gmax = ag;
            if (sm.v[i] != F(0)) vzero = false;
        }
        for (int off = 16; off; off >>= 1) gmax = fmax(gmax, __shfl_xor_sync(PS_FULL, gmax, off));
        vzero = __all_sync(PS_FULL, vzero);
        if (gmax < F(1e-12)) {
            frozen = true;
            continue;
        }
        bool fresh = vzero;
        for (int i = lane; i < n; i += 32) sm.v[i] = momentum * sm.v[i] - sm.g[i];
        __syncwarp();
        F dd = 0;
        if (lane == 0)
            for (int i = 0; i < n; ++i) dd += sm.g[i] * sm.v[i];
        dd = __shfl_sync(PS_FULL, dd, 0);
        if (dd >= F(0)) {
            fresh = true;
            for (int i = lane; i < n; i += 32) sm.v[i] = -sm.g[i];
            __syncwarp();
            dd = 0;
            if (lane == 0)
                for (int i = 0; i < n; ++i) dd -= sm.g[i] * sm.g[i];
            dd = __shfl_sync(PS_FULL, dd, 0);
        }
        F a = alpha * F(2.0);
        if (a > alpha_max) a = alpha_max;
        bool accepted = false;
        F fc = 0;
        for (int bt = 0; bt < max_backtracks; ++bt) {
            for (int i = lane; i < n; i += 32) sm.cand[i] = sm.q[i] + a * sm.v[i];
            __syncwarp();
            int clc;
            F totc = seed_cost(A, sm.cand, T, false, sm.sc, sm.g + 0 /*unused*/, sm.terms, clc);
            fc = clc ? INF : totc;
            if (fc <= f + armijo_c * a * dd) {
                accepted = true;
                break;
            }
            a *= shrink;
        }
        if (accepted) {
            for (int i = lane; i < n; i += 32) sm.q[i] = sm.q[i] + a * sm.v[i];
            f = fc;
            alpha = a;
            n_acc += 1;
        } else {
            for (int i = lane; i < n; i += 32) sm.v[i] = 0;
            if (fresh) frozen = true;
        }
        __syncwarp();
    }
    const F tot = seed_cost(A, sm.q, T, false, sm.sc, sm.g, sm.terms, cl);
    for (int i = lane; i < n; i += 32) x_out[(size_t)s * n + i] = sm.q[i];
    if (lane == 0) {
        for (int i = 0; i < 5; ++i) terms_out[s * 5 + i] = sm.terms[i];
        totals[s] = tot;
        frozen_out[s] = frozen ? 1 : 0;
        n_acc_out[s] = n_acc;
    }
}

// ---------------------------------------------------------------------------
// Cost guidance of one DDIM sub-step (guided_ddim_sample's `guide`, src/diffusion.py:598-617),
// fused for the planner cost (evaluate_cost_batch, src/trajopt.py:105-119).  One warp per
// seed, all seeds in one cooperative grid: the reference evaluates the whole batch at every
// halving while ANY seed still backtracks (phantom candidates of finished seeds included),
// and raises at the first evaluation that leaves the ESDF, so each evaluation ends in a grid
// barrier that exchanges {clamped, remaining} over all seeds.
//   x (S,T,D) normalised x0_hat, updated in place; q = arm_lo + x * arm_span (arm.denormalize);
//   g_norm = grad * net_span; cand = x - step * g_norm.
//   flags: 2*S ints (double-buffered exchange); err: 2 + S ints
//   (err[0] = 1 if an evaluation was clamped, err[1] = its index, err[2+s] = seed s clamped).
// ---------------------------------------------------------------------------
template <typename F>
__global__ void __launch_bounds__(32) guide_kernel(const __grid_constant__ ArmGrid<F> A, F* __restrict__ x, int S,
                                                   int T, const F* __restrict__ arm_lo,
                                                   const F* __restrict__ arm_span, const F* __restrict__ net_span,
                                                   int n_grad, F alpha_guide, int max_halvings,
                                                   int* __restrict__ flags, int* __restrict__ err) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) uint8_t smraw[];
    SeedSmem<F>& sm = *reinterpret_cast<SeedSmem<F>*>(smraw);
    const int s = blockIdx.x, lane = threadIdx.x;
    const int D = A.D, n = T * D;
    F* xs = sm.q;      // x (normalised)
    F* gn = sm.v;      // g_norm
    F* cx = sm.cand;   // candidate (normalised)
    F* qd = sm.g;      // denormalised evaluation point; later the cost gradient
    __shared__ F grad_buf[MAXT * MAXD];
    for (int i = lane; i < n; i += 32) xs[i] = x[(size_t)s * n + i];
    if (s == 0 && lane == 0) err[0] = 0;
    __syncwarp();
    int n_eval = 0;
    // exchange: publish (remaining | clamped<<1), barrier, OR over all seeds
    auto exchange = [&](bool remaining, bool clamped, bool& any_rem, bool& any_cl) {
        int* buf = flags + (n_eval & 1) * S;
        if (lane == 0) buf[s] = (remaining ? 1 : 0) | (clamped ? 2 : 0);
        __threadfence();
        grid.sync();
        int acc = 0;
        for (int j = lane; j < S; j += 32) acc |= __ldcg(buf + j);
        for (int off = 16; off; off >>= 1) acc |= __shfl_xor_sync(PS_FULL, acc, off);
        any_rem = (acc & 1) != 0;
        any_cl = (acc & 2) != 0;
        if (any_cl && s == 0) {
            for (int j = lane; j < S; j += 32) err[2 + j] = (__ldcg(buf + j) & 2) ? 1 : 0;
            if (lane == 0) {
                err[1] = n_eval;
                err[0] = 1;
            }
        }
        ++n_eval;
    };
    for (int it = 0; it < n_grad; ++it) {
        for (int i = lane; i < n; i += 32) qd[i] = arm_lo[i % D] + xs[i] * arm_span[i % D];
        __syncwarp();
        int cl;
        const F cost = seed_cost(A, qd, T, true, sm.sc, grad_buf, sm.terms, cl);
        __syncwarp();
        bool any_rem, any_cl;
        exchange(true, cl != 0, any_rem, any_cl);
        if (any_cl) return;
        for (int i = lane; i < n; i += 32) gn[i] = grad_buf[i] * net_span[i % D];
        __syncwarp();
        F step = alpha_guide;
        bool remaining = true;
        any_rem = true;
        for (int h = 0; h < max_halvings; ++h) {
            if (!any_rem) break;
            for (int i = lane; i < n; i += 32) {
                cx[i] = xs[i] - step * gn[i];
                qd[i] = arm_lo[i % D] + cx[i] * arm_span[i % D];
            }
            __syncwarp();
            int clc;
            const F nc = seed_cost(A, qd, T, true, sm.sc, grad_buf, sm.terms, clc);
            __syncwarp();
            const bool improved = remaining && (nc < cost);
            if (improved)
                for (int i = lane; i < n; i += 32) xs[i] = cx[i];
            remaining = remaining && !improved;
            if (remaining) step = step * F(0.5);
            __syncwarp();
            exchange(remaining, clc != 0, any_rem, any_cl);
            if (any_cl) return;
        }
    }
    for (int i = lane; i < n; i += 32) x[(size_t)s * n + i] = xs[i];
}

// x = sqrt(ab_next) * x0 + sqrt(1 - ab_next) * eps (the DDIM step after guidance, src/diffusion.py:553-555)
__global__ void ddim_next_kernel(double* __restrict__ x, const double* __restrict__ x0,
                                 const double* __restrict__ eps, int n, double ab_next) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    x[i] = sqrt(ab_next) * x0[i] + sqrt(1.0 - ab_next) * eps[i];
}

// ---------------------------------------------------------------------------
// Ground-truth trajectory metrics (trajopt.metrics / retime, src/trajopt.py:209-272;
// _kernels.analytic_sdf / config_clearance / traj_min_clearance, src/_kernels.py:60-162).
// One warp per trajectory: lanes stride over the T + (T-1)*interp configurations for the
// analytic clearance (min is order-independent), then the end pose, the retime scale from
// the numpy.gradient stencils (products by +-0.5/1 are exact, so v, a, j are bit-exact)
// and max |J q| / dt^3.
// ---------------------------------------------------------------------------
struct GTWorld {
    const double* circles;   // (nc, 3): cx, cy, r
    const double* boxes;     // (nb, 4): lox, loy, hix, hiy
    int nc, nb;
    double cap;
};

__device__ double analytic_sdf(const GTWorld& W, double x, double y) {
    double best = W.cap;
    for (int k = 0; k < W.nc; ++k) {
        const double dx = x - W.circles[3 * k], dy = y - W.circles[3 * k + 1];
        const double d = sqrt(dx * dx + dy * dy) - W.circles[3 * k + 2];
        if (d < best) best = d;
    }
    for (int k = 0; k < W.nb; ++k) {
        const double* b = W.boxes + 4 * k;
        const double cx = 0.5 * (b[0] + b[2]), cy = 0.5 * (b[1] + b[3]);
        const double qx = fabs(x - cx) - 0.5 * (b[2] - b[0]);
        const double qy = fabs(y - cy) - 0.5 * (b[3] - b[1]);
        const double ax = qx > 0.0 ? qx : 0.0, ay = qy > 0.0 ? qy : 0.0;
        double inside = qx > qy ? qx : qy;
        if (inside > 0.0) inside = 0.0;
        const double d = sqrt(ax * ax + ay * ay) + inside;
        if (d < best) best = d;
    }
    return best;
}

__device__ double config_clearance(const ArmGrid<double>& A, const GTWorld& W, const double* q) {
    double best = W.cap, th = 0.0, px = A.basex, py = A.basey;
    for (int k = 0; k < A.D; ++k) {
        th += q[k];
        const double c = cos(th), s = sin(th);
        for (int i = 0; i < A.M; ++i) {
            const double x = px + A.fracs[i] * A.lengths[k] * c;
            const double y = py + A.fracs[i] * A.lengths[k] * s;
            const double v = analytic_sdf(W, x, y);
            if (v < best) best = v;
        }
        px += A.lengths[k] * c;
        py += A.lengths[k] * s;
    }
    return best;
}

__global__ void __launch_bounds__(32) metrics_kernel(const __grid_constant__ ArmGrid<double> A, const GTWorld W,
                                                     const double* __restrict__ trajs, int S, int T, int interp,
                                                     const double* __restrict__ vel, const double* __restrict__ acc,
                                                     const double* __restrict__ jerk, double* __restrict__ out) {
    __shared__ double q[MAXT * MAXD], v[MAXT * MAXD], a[MAXT * MAXD], j[MAXT * MAXD];
    const int s = blockIdx.x, lane = threadIdx.x, D = A.D, n = T * D;
    const double* tr = trajs + (size_t)s * n;
    for (int i = lane; i < n; i += 32) q[i] = tr[i];
    __syncwarp();
    // clearance over waypoints + interpolants (traj_min_clearance)
    const int per = interp + 1, n_cfg = (T - 1) * per + 1;
    double best = W.cap;
    for (int c = lane; c < n_cfg; c += 32) {
        const int t = c / per, i = c % per;
        double qc[MAXD];
        if (i == 0) {
            for (int k = 0; k < D; ++k) qc[k] = q[t * D + k];
        } else {
            const double f = (double)i / (double)per;
            for (int k = 0; k < D; ++k) qc[k] = q[t * D + k] + f * (q[(t + 1) * D + k] - q[t * D + k]);
        }
        const double cv = config_clearance(A, W, qc);
        if (cv < best) best = cv;
    }
    for (int off = 16; off; off >>= 1) best = fmin(best, __shfl_xor_sync(PS_FULL, best, off));
    // numpy.gradient stencil applied three times (diff_matrix, src/trajopt.py:64-73)
    auto grad1 = [&](const double* x, double* y) {
        for (int idx = lane; idx < n; idx += 32) {
            const int r = idx / D, k = idx % D;
            double val;
            if (r == 0) val = -1.0 * x[k] + 1.0 * x[D + k];
            else if (r == T - 1) val = -1.0 * x[(T - 2) * D + k] + 1.0 * x[(T - 1) * D + k];
            else val = -0.5 * x[(r - 1) * D + k] + 0.5 * x[(r + 1) * D + k];
            y[idx] = val;
        }
        __syncwarp();
    };
    grad1(q, v);
    grad1(v, a);
    grad1(a, j);
    // dt = max(max(vmax/vl), sqrt(max(amax/al)), cbrt(max(jmax/jl))) (retime, src/trajopt.py:209-229)
    double rv = 0.0, ra = 0.0, rj = 0.0;
    if (lane < D) {
        double vm = 0.0, am = 0.0, jm = 0.0;
        for (int r = 0; r < T; ++r) {
            vm = fmax(vm, fabs(v[r * D + lane]));
            am = fmax(am, fabs(a[r * D + lane]));
            jm = fmax(jm, fabs(j[r * D + lane]));
        }
        rv = vm / vel[lane];
        ra = am / acc[lane];
        rj = jm / jerk[lane];
    }
    for (int off = 16; off; off >>= 1) {
        rv = fmax(rv, __shfl_xor_sync(PS_FULL, rv, off));
        ra = fmax(ra, __shfl_xor_sync(PS_FULL, ra, off));
        rj = fmax(rj, __shfl_xor_sync(PS_FULL, rj, off));
    }
    const double dt = fmax(fmax(rv, sqrt(ra)), cbrt(rj));
    const double motion_time = dt * (double)(T - 1);
    // max |jerk_matrix @ traj| / dt^3 (dense J as the reference forms it)
    double mj = 0.0;
    for (int idx = lane; idx < n; idx += 32) {
        const int r = idx / D, k = idx % D;
        double y = 0.0;
        for (int c = 0; c < T; ++c) y += A.jerk_mat[r * T + c] * q[c * D + k];
        mj = fmax(mj, fabs(y));
    }
    for (int off = 16; off; off >>= 1) mj = fmax(mj, __shfl_xor_sync(PS_FULL, mj, off));
    if (lane == 0) {
        // end pose (fk_pose, src/arm.py:118-125) and its errors against the goal
        double th = 0.0, ex = A.basex, ey = A.basey;
        const double* qe = q + (T - 1) * D;
        for (int k = 0; k < D; ++k) {
            th += qe[k];
            ex += A.lengths[k] * cos(th);
            ey += A.lengths[k] * sin(th);
        }
        const double pi = 3.141592653589793238462643383279502884;
        const double end_th = wrap(th);
        const double terr = hypot(ex - A.goal_x, ey - A.goal_y);
        const double aerr = fabs(wrap(end_th - A.goal_th)) * (180.0 / pi);
        double* o = out + (size_t)s * 6;
        o[0] = best;
        o[1] = terr;
        o[2] = aerr;
        o[3] = motion_time;
        o[4] = motion_time > 0.0 ? mj / (dt * dt * dt) : 0.0;
        o[5] = dt;
    }
}

// ---------------------------------------------------------------------------
// Observation synthesis: geometry.render_depth_scan / _ray_hits (src/geometry.py:279-329),
// one thread per ray, the reference's expressions in the reference's order (fp64).
// ---------------------------------------------------------------------------
__global__ void render_scan_kernel(const double* __restrict__ circles, int nc, const double* __restrict__ boxes,
                                   int nb, double px, double py, double heading, double fov, int n_rays,
                                   double max_range, double* __restrict__ depths) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rays) return;
    // pose.ray_angles(): heading + np.linspace(-fov/2, fov/2, n_rays)
    const double start = -fov / 2, stop = fov / 2;
    const double step = (stop - start) / (double)(n_rays - 1);
    const double lin = (i == n_rays - 1) ? stop : (double)i * step + start;
    const double ang = heading + lin;
    const double dx = cos(ang), dy = sin(ang);
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    double t_best = max_range;
    if (nc > 0) {
        double tmin = inf;
        for (int k = 0; k < nc; ++k) {
            const double mx = circles[3 * k] - px, my = circles[3 * k + 1] - py, r = circles[3 * k + 2];
            const double b = dx * mx + dy * my;
            const double cc = mx * mx + my * my - r * r;
            const double disc = b * b - cc;
            const bool ok = disc >= 0;
            const double sq = sqrt(ok ? disc : 0.0);
            double t1 = b - sq, t2 = b + sq;
            t1 = (ok && t1 > 1e-12) ? t1 : inf;
            t2 = (ok && t2 > 1e-12) ? t2 : inf;
            tmin = fmin(tmin, fmin(t1, t2));
        }
        t_best = fmin(t_best, tmin);
    }
    if (nb > 0) {
        double tmin = inf;
        const bool par_x = fabs(dx) < 1e-300, par_y = fabs(dy) < 1e-300;
        for (int k = 0; k < nb; ++k) {
            const double* bx = boxes + 4 * k;
            const double tx1 = (bx[0] - px) / dx, tx2 = (bx[2] - px) / dx;
            const double ty1 = (bx[1] - py) / dy, ty2 = (bx[3] - py) / dy;
            const bool in_x = (px >= bx[0]) && (px <= bx[2]);
            const bool in_y = (py >= bx[1]) && (py <= bx[3]);
            const double tx_lo = par_x ? (in_x ? -inf : inf) : fmin(tx1, tx2);
            const double tx_hi = par_x ? (in_x ? inf : -inf) : fmax(tx1, tx2);
            const double ty_lo = par_y ? (in_y ? -inf : inf) : fmin(ty1, ty2);
            const double ty_hi = par_y ? (in_y ? inf : -inf) : fmax(ty1, ty2);
            const double t_near = fmax(tx_lo, ty_lo), t_far = fmin(tx_hi, ty_hi);
            const bool hit = t_near <= t_far;
            double t = t_near > 1e-12 ? t_near : t_far;   // origin inside -> exit point
            t = (hit && t > 1e-12) ? t : inf;
            tmin = fmin(tmin, t);
        }
        t_best = fmin(t_best, tmin);
    }
    depths[i] = fmin(t_best, max_range);
}

// ---------------------------------------------------------------------------
// scan-derived planner ESDF (src/pipeline.py:101-132; geometry.py:130-152, :270-276)
// ---------------------------------------------------------------------------
__global__ void planner_esdf_kernel(const double* __restrict__ depths, int n_rays, double sx, double sy,
                                    double heading, double fov, double max_range, double r_disc, double cap,
                                    double ox, double oy, double h, int nx, int ny, double* __restrict__ out) {
    __shared__ double cx[1024], cy[1024];
    __shared__ int n_hit;
    if (threadIdx.x == 0) {
        // np.linspace(-fov/2, fov/2, n) then hit filter (depth < max_range - 1e-9), in ray order
        int m = 0;
        const double start = -fov / 2, stop = fov / 2;
        const double step = (stop - start) / (double)(n_rays - 1);
        for (int i = 0; i < n_rays && m < 1024; ++i) {
            const double d = depths[i];
            if (d < max_range - 1e-9) {
                const double lin = (i == n_rays - 1) ? stop : start + (double)i * step;
                const double ang = heading + lin;
                cx[m] = sx + d * cos(ang);
                cy[m] = sy + d * sin(ang);
                ++m;
            }
        }
        n_hit = m;
    }
    __syncthreads();
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nx * ny) return;
    const int i = idx / ny, j = idx % ny;
    const double x = ox + h * (double)i, y = oy + h * (double)j;
    double best = cap;
    if (n_hit > 0) {
        double mn = INFINITY;
        for (int k = 0; k < n_hit; ++k) {
            const double dc = hypot(x - cx[k], y - cy[k]) - r_disc;
            mn = fmin(mn, dc);
        }
        best = fmin(best, mn);
    }
    out[idx] = best;
}

// planner_success (src/pipeline.py:139-157): one thread per seed.
__global__ void planner_success_kernel(const __grid_constant__ ArmGrid<double> A, const double* __restrict__ trajs,
                                       int S, int T, double delta_t, double delta_r_deg, int interp,
                                       uint8_t* __restrict__ ok) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const int D = A.D, M = A.M;
    const double* tr = trajs + (size_t)s * T * D;
    double dmin = INFINITY;
    for (int f = 0; f <= interp; ++f) {
        const double fr = f == 0 ? 0.0 : (double)f / (double)(interp + 1);
        const int rows = f == 0 ? T : T - 1;
        for (int t = 0; t < rows; ++t) {
            double q[MAXD], th = 0, lx[MAXD], ly[MAXD], cx = 0, cy = 0;
            for (int k = 0; k < D; ++k) q[k] = f == 0 ? tr[t * D + k] : tr[t * D + k] + fr * (tr[(t + 1) * D + k] - tr[t * D + k]);
            for (int k = 0; k < D; ++k) {
                th += q[k];
                lx[k] = A.lengths[k] * cos(th);
                ly[k] = A.lengths[k] * sin(th);
            }
            for (int k = 0; k < D; ++k) {
                cx += lx[k];
                cy += ly[k];
                const double prex = cx - lx[k], prey = cy - ly[k];  // cumsum(lx) - lx
                for (int i = 0; i < M; ++i) {
                    const double px = A.basex + prex + A.fracs[i] * lx[k];
                    const double py = A.basey + prey + A.fracs[i] * ly[k];
                    double d, gx, gy;
                    bool cl;
                    bilinear(A, px, py, d, gx, gy, cl);
                    dmin = fmin(dmin, d);
                }
            }
        }
    }
    bool good = dmin > 0.0;
    if (good) {
        double th = 0, x = 0, y = 0;
        for (int k = 0; k < D; ++k) {
            th += tr[(T - 1) * D + k];
            x += A.lengths[k] * cos(th);
            y += A.lengths[k] * sin(th);
        }
        x += A.basex;
        y += A.basey;
        const double terr = hypot(x - A.goal_x, y - A.goal_y);
        const double aerr = fabs(wrap(th - A.goal_th)) * (180.0 / 3.141592653589793238462643383279502884);
        good = terr <= delta_t && aerr <= delta_r_deg;
    }
    ok[s] = good ? 1 : 0;
}

// ---------------------------------------------------------------------------
// FC denoiser (src/diffusion.py:272-300) and scan encoder (:246-269), fp64
// ---------------------------------------------------------------------------
// Templated on the scalar type: float64 is planseed's parity mode, float32 the fast mode
// (SURVEY §7.2); the arithmetic is the same expression in either type.
template <typename F>
__device__ __forceinline__ F silu(F x) { return x * (F(1) / (F(1) + exp(-x))); }

// y[r, n] = act(b[n] + sum_k x[r, k] W[k, n]); W (K, N) row-major ("in, out")
template <typename F>
__global__ void linear_kernel(const F* __restrict__ x, int ldx, const F* __restrict__ W, const F* __restrict__ b,
                              int R, int K, int N, int act, F* __restrict__ y, int ldy) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
    if (n >= N || r >= R) return;
    F acc = 0;
    const F* xr = x + (size_t)r * ldx;
    for (int k = 0; k < K; ++k) acc += xr[k] * W[(size_t)k * N + n];
    acc += b[n];
    y[(size_t)r * ldy + n] = act ? silu(acc) : acc;
}

// h = h * (1 + scale) + shift, scale/shift rows broadcast (mod is shared by the batch)
template <typename F>
__global__ void film_kernel(F* __restrict__ h, const F* __restrict__ scale, const F* __restrict__ shift, int R,
                            int N) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
    if (n >= N || r >= R) return;
    F& v = h[(size_t)r * N + n];
    v = v * (F(1) + scale[n]) + shift[n];
}

// conv1d valid, stride s: (C_in, L) x (C_out, C_in, K) -> silu -> (C_out, Lo); one block
template <typename F>
__global__ void conv1d_silu_kernel(const F* __restrict__ x, int C, int L, const F* __restrict__ w,
                                   const F* __restrict__ b, int O, int Kk, int stride, F* __restrict__ y) {
    const int Lo = (L - Kk) / stride + 1;
    for (int idx = threadIdx.x; idx < O * Lo; idx += blockDim.x) {
        const int o = idx / Lo, j = idx % Lo;
        F acc = 0;
        for (int c = 0; c < C; ++c)
            for (int t = 0; t < Kk; ++t) acc += w[((size_t)o * C + c) * Kk + t] * x[(size_t)c * L + j * stride + t];
        y[idx] = silu(acc + b[o]);
    }
}

// DDIM update (src/diffusion.py:547-555) on the normalised state; the schedule coefficients are
// formed in float64 on the host and rounded once to F
template <typename F>
__global__ void ddim_update_kernel(F* __restrict__ x, const F* __restrict__ eps, int n, F sq1m, F rsq, F sqn,
                                   F sq1mn, int has_next, F clip_lo, F clip_hi, F* __restrict__ x0_out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    F x0 = (x[i] - sq1m * eps[i]) / rsq;
    x0 = fmin(fmax(x0, clip_lo), clip_hi);
    x0_out[i] = x0;
    if (has_next) x[i] = sqn * x0 + sq1mn * eps[i];
}

}  // namespace ref
}  // namespace ps

using namespace ps;
using namespace ps::ref;

template <typename F>
static int fill_arm(ArmGrid<F>& A, int D, const double* lengths_h, double basex, double basey, const double* fracs_h,
                    int M, const long long* pa_h, const long long* pb_h, int n_pairs, const void* grid, int nx,
                    int ny, double gox, double goy, double gh, double goal_x, double goal_y, double goal_th,
                    const double* w_h, double d_act, double d_self, const void* jm, const void* jq) {
    if (D < 1 || D > MAXD || M < 1 || M > MAXM || n_pairs < 0 || n_pairs > MAXPAIR || nx < 2 || ny < 2)
        return PS_FAIL(PS_ERR_SHAPE);
    A.D = D;
    A.M = M;
    A.n_pairs = n_pairs;
    for (int k = 0; k < D; ++k) A.lengths[k] = (F)lengths_h[k];
    for (int i = 0; i < M; ++i) A.fracs[i] = (F)fracs_h[i];
    A.basex = (F)basex;
    A.basey = (F)basey;
    for (int e = 0; e < n_pairs; ++e) {
        if (pa_h[e] < 0 || pa_h[e] >= D * M || pb_h[e] < 0 || pb_h[e] >= D * M) return PS_FAIL(PS_ERR_SHAPE);
        A.pair_a[e] = (short)pa_h[e];
        A.pair_b[e] = (short)pb_h[e];
    }
    A.grid = reinterpret_cast<const F*>(grid);
    A.nx = nx;
    A.ny = ny;
    A.gox = (F)gox;
    A.goy = (F)goy;
    A.gh = (F)gh;
    A.goal_x = (F)goal_x;
    A.goal_y = (F)goal_y;
    A.goal_th = (F)goal_th;
    for (int i = 0; i < 5; ++i) A.w[i] = (F)w_h[i];
    A.d_act = (F)d_act;
    A.d_self = (F)d_self;
    A.jerk_mat = reinterpret_cast<const F*>(jm);
    A.jerk_quad = reinterpret_cast<const F*>(jq);
    return PS_OK;
}

#define REF_ARM_ARGS                                                                                             \
    const double *lengths_h, double basex, double basey, const double *fracs_h, int M, const long long *pair_a_h, \
        const long long *pair_b_h, int n_pairs, const void *grid, int nx, int ny, double gox, double goy,         \
        double gh, double goal_x, double goal_y, double goal_th, const double *weights_h, double d_act,          \
        double d_self, const void *jerk_mat, const void *jerk_quad
#define REF_ARM_PASS                                                                                            \
    lengths_h, basex, basey, fracs_h, M, pair_a_h, pair_b_h, n_pairs, grid, nx, ny, gox, goy, gh, goal_x, goal_y, \
        goal_th, weights_h, d_act, d_self, jerk_mat, jerk_quad

template <typename F>
static int ref_cost(const void* qs, int S, int T, int D, REF_ARM_ARGS, int want_grad, void* terms, void* totals,
                    void* grads, uint8_t* clamped, cudaStream_t st) {
    ArmGrid<F> A;
    int e = fill_arm(A, D, REF_ARM_PASS);
    if (e) return e;
    if (T < 2 || T > MAXT || S < 0) return PS_FAIL(PS_ERR_SHAPE);
    if (S == 0) return PS_OK;
    const size_t smem = sizeof(SeedSmem<F>);
    auto k = cost_kernel<F>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<S, 32, smem, st>>>(A, (const F*)qs, S, T, want_grad, (F*)terms, (F*)totals, (F*)grads, clamped);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

template <typename F>
static int ref_opt(const void* seeds, int S, int T, int D, int n_iters, double momentum, double armijo_c,
                   double shrink, int max_bt, double alpha0, double alpha_max, REF_ARM_ARGS, void* x_out, void* terms,
                   void* totals, uint8_t* frozen, long long* n_acc, cudaStream_t st) {
    ArmGrid<F> A;
    int e = fill_arm(A, D, REF_ARM_PASS);
    if (e) return e;
    if (T < 2 || T > MAXT || S < 0 || n_iters < 0) return PS_FAIL(PS_ERR_SHAPE);
    if (S == 0) return PS_OK;
    const size_t smem = sizeof(SeedSmem<F>);
    auto k = optimize_kernel<F>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<S, 32, smem, st>>>(A, (const F*)seeds, S, T, n_iters, (F)momentum, (F)armijo_c, (F)shrink, max_bt, (F)alpha0,
                           (F)alpha_max, (F*)x_out, (F*)terms, (F*)totals, frozen, n_acc);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

template <typename F>
static int ref_guide(void* x, int S, int T, int D, REF_ARM_ARGS, const double* arm_lo_d, const double* arm_span_d,
                     const double* net_span_d, int n_grad, double alpha_guide, int max_halvings, int* flags, int* err,
                     cudaStream_t st) {
    ArmGrid<F> A;
    int e = fill_arm(A, D, REF_ARM_PASS);
    if (e) return e;
    if (T < 2 || T > MAXT || S < 0 || n_grad < 0 || max_halvings < 0) return PS_FAIL(PS_ERR_SHAPE);
    if (S == 0 || n_grad == 0) return PS_OK;
    const size_t smem = sizeof(SeedSmem<F>);
    auto k = guide_kernel<F>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0, dev = 0, n_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32, smem);
    if ((long long)per_sm * n_sm < S) return PS_FAIL(PS_ERR_SHAPE);  // all seeds must be co-resident
    F* xp = (F*)x;
    const F* lo = (const F*)arm_lo_d;
    const F* sp = (const F*)arm_span_d;
    const F* ns = (const F*)net_span_d;
    F ag = (F)alpha_guide;
    void* args[] = {(void*)&A, (void*)&xp, (void*)&S, (void*)&T, (void*)&lo, (void*)&sp, (void*)&ns,
                    (void*)&n_grad, (void*)&ag, (void*)&max_halvings, (void*)&flags, (void*)&err};
    ps_launch_counter().fetch_add(1, std::memory_order_relaxed);
    if (cudaLaunchCooperativeKernel((const void*)k, dim3(S), dim3(32), args, smem, st) != cudaSuccess)
        return PS_FAIL(PS_ERR_CUDA);
    return PS_OK;
}

extern "C" int ps_ref_guide(int dtype, void* x, int S, int T, int D, REF_ARM_ARGS, const void* arm_lo,
                            const void* arm_span, const void* net_span, int n_grad, double alpha_guide,
                            int max_halvings, int* flags, int* err, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == 0)
        return ref_guide<double>(x, S, T, D, REF_ARM_PASS, (const double*)arm_lo, (const double*)arm_span,
                                 (const double*)net_span, n_grad, alpha_guide, max_halvings, flags, err, st);
    if (dtype == 1)
        return ref_guide<float>(x, S, T, D, REF_ARM_PASS, (const double*)arm_lo, (const double*)arm_span,
                                (const double*)net_span, n_grad, alpha_guide, max_halvings, flags, err, st);
    return PS_FAIL(PS_ERR_SHAPE);
}

extern "C" int ps_ref_metrics(const double* trajs, int S, int T, int D, const double* lengths_h, double basex,
                              double basey, const double* fracs_h, int M, const double* circles, int nc,
                              const double* boxes, int nb, double cap, double goal_x, double goal_y, double goal_th,
                              const double* jerk_mat, const double* vel, const double* acc, const double* jerk,
                              int interp, double* out, void* stream) {
    if (D < 1 || D > MAXD || M < 1 || M > MAXM || T < 2 || T > MAXT || S < 0 || interp < 0 || nc < 0 || nb < 0)
        return PS_FAIL(PS_ERR_SHAPE);
    if (S == 0) return PS_OK;
    ArmGrid<double> A{};
    A.D = D;
    A.M = M;
    for (int k = 0; k < D; ++k) A.lengths[k] = lengths_h[k];
    for (int i = 0; i < M; ++i) A.fracs[i] = fracs_h[i];
    A.basex = basex;
    A.basey = basey;
    A.goal_x = goal_x;
    A.goal_y = goal_y;
    A.goal_th = goal_th;
    A.jerk_mat = jerk_mat;
    GTWorld W{circles, boxes, nc, nb, cap};
    metrics_kernel<<<S, 32, 0, (cudaStream_t)stream>>>(A, W, trajs, S, T, interp, vel, acc, jerk, out);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_ref_ddim_next(double* x, const double* x0, const double* eps, int n, double ab_next,
                                void* stream) {
    if (n <= 0) return PS_FAIL(PS_ERR_SHAPE);
    ddim_next_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(x, x0, eps, n, ab_next);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_ref_cost_terms(int dtype, const void* qs, int S, int T, int D, REF_ARM_ARGS, int want_grad,
                                 void* terms, void* totals, void* grads, uint8_t* clamped, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == 0)
        return ref_cost<double>(qs, S, T, D, REF_ARM_PASS, want_grad, terms, totals, grads, clamped, st);
    if (dtype == 1)
        return ref_cost<float>(qs, S, T, D, REF_ARM_PASS, want_grad, terms, totals, grads, clamped, st);
    return PS_FAIL(PS_ERR_SHAPE);
}

extern "C" int ps_ref_optimize(int dtype, const void* seeds, int S, int T, int D, int n_iters, double momentum,
                               double armijo_c, double shrink, int max_backtracks, double alpha0, double alpha_max,
                               REF_ARM_ARGS, void* x_out, void* terms, void* totals, uint8_t* frozen,
                               long long* n_accepted, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == 0)
        return ref_opt<double>(seeds, S, T, D, n_iters, momentum, armijo_c, shrink, max_backtracks, alpha0, alpha_max,
                               REF_ARM_PASS, x_out, terms, totals, frozen, n_accepted, st);
    if (dtype == 1)
        return ref_opt<float>(seeds, S, T, D, n_iters, momentum, armijo_c, shrink, max_backtracks, alpha0, alpha_max,
                              REF_ARM_PASS, x_out, terms, totals, frozen, n_accepted, st);
    return PS_FAIL(PS_ERR_SHAPE);
}

extern "C" int ps_ref_render_scan(const double* circles, int nc, const double* boxes, int nb, double px, double py,
                                  double heading, double fov, int n_rays, double max_range, double* depths,
                                  void* stream) {
    if (n_rays < 2 || nc < 0 || nb < 0) return PS_FAIL(PS_ERR_SHAPE);
    render_scan_kernel<<<(n_rays + 127) / 128, 128, 0, (cudaStream_t)stream>>>(circles, nc, boxes, nb, px, py,
                                                                                heading, fov, n_rays, max_range,
                                                                                depths);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_ref_planner_esdf(const double* depths, int n_rays, double sx, double sy, double heading, double fov,
                                   double max_range, double r_disc, double cap, double ox, double oy, double h,
                                   int nx, int ny, double* out, void* stream) {
    if (n_rays < 2 || n_rays > 1024 || nx < 2 || ny < 2) return PS_FAIL(PS_ERR_SHAPE);
    const int n = nx * ny;
    planner_esdf_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
        depths, n_rays, sx, sy, heading, fov, max_range, r_disc, cap, ox, oy, h, nx, ny, out);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_ref_planner_success(const double* trajs, int S, int T, int D, REF_ARM_ARGS, double delta_t,
                                      double delta_r_deg, int interp, uint8_t* ok, void* stream) {
    ArmGrid<double> A;
    int e = fill_arm(A, D, REF_ARM_PASS);
    if (e) return e;
    if (S == 0) return PS_OK;
    planner_success_kernel<<<(S + 63) / 64, 64, 0, (cudaStream_t)stream>>>(A, trajs, S, T, delta_t, delta_r_deg,
                                                                            interp, ok);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

// dtype: 0 float64 (parity mode), 1 float32 (fast mode); pointers of that type
extern "C" int ps_ref_linear_dt(int dtype, const void* x, int ldx, const void* W, const void* b, int R, int K, int N,
                                int act, void* y, int ldy, void* stream) {
    if (R <= 0 || K <= 0 || N <= 0 || (dtype != 0 && dtype != 1)) return PS_FAIL(PS_ERR_SHAPE);
    const dim3 g((N + 127) / 128, R);
    if (dtype == 0)
        linear_kernel<double><<<g, 128, 0, (cudaStream_t)stream>>>((const double*)x, ldx, (const double*)W,
                                                                    (const double*)b, R, K, N, act, (double*)y, ldy);
    else
        linear_kernel<float><<<g, 128, 0, (cudaStream_t)stream>>>((const float*)x, ldx, (const float*)W,
                                                                   (const float*)b, R, K, N, act, (float*)y, ldy);
    PS_CHECK_LAUNCH();
    return PS_OK;
}
extern "C" int ps_ref_linear(const double* x, int ldx, const double* W, const double* b, int R, int K, int N, int act,
                             double* y, int ldy, void* stream) {
    return ps_ref_linear_dt(0, x, ldx, W, b, R, K, N, act, y, ldy, stream);
}

extern "C" int ps_ref_film_dt(int dtype, void* h, const void* scale, const void* shift, int R, int N, void* stream) {
    if (R <= 0 || N <= 0 || (dtype != 0 && dtype != 1)) return PS_FAIL(PS_ERR_SHAPE);
    const dim3 g((N + 127) / 128, R);
    if (dtype == 0)
        film_kernel<double><<<g, 128, 0, (cudaStream_t)stream>>>((double*)h, (const double*)scale,
                                                                  (const double*)shift, R, N);
    else
        film_kernel<float><<<g, 128, 0, (cudaStream_t)stream>>>((float*)h, (const float*)scale, (const float*)shift,
                                                                 R, N);
    PS_CHECK_LAUNCH();
    return PS_OK;
}
extern "C" int ps_ref_film(double* h, const double* scale, const double* shift, int R, int N, void* stream) {
    return ps_ref_film_dt(0, h, scale, shift, R, N, stream);
}

extern "C" int ps_ref_conv1d_silu_dt(int dtype, const void* x, int C, int L, const void* w, const void* b, int O,
                                     int K, int stride, void* y, void* stream) {
    if (L < K || (dtype != 0 && dtype != 1)) return PS_FAIL(PS_ERR_SHAPE);
    if (dtype == 0)
        conv1d_silu_kernel<double><<<1, 256, 0, (cudaStream_t)stream>>>((const double*)x, C, L, (const double*)w,
                                                                         (const double*)b, O, K, stride, (double*)y);
    else
        conv1d_silu_kernel<float><<<1, 256, 0, (cudaStream_t)stream>>>((const float*)x, C, L, (const float*)w,
                                                                        (const float*)b, O, K, stride, (float*)y);
    PS_CHECK_LAUNCH();
    return PS_OK;
}
extern "C" int ps_ref_conv1d_silu(const double* x, int C, int L, const double* w, const double* b, int O, int K,
                                  int stride, double* y, void* stream) {
    return ps_ref_conv1d_silu_dt(0, x, C, L, w, b, O, K, stride, y, stream);
}

extern "C" int ps_ref_ddim_update_dt(int dtype, void* x, const void* eps, int n, double ab, double ab_next,
                                     int has_next, double clip_lo, double clip_hi, void* x0_out, void* stream) {
    if (n <= 0 || (dtype != 0 && dtype != 1)) return PS_FAIL(PS_ERR_SHAPE);
    const double sq1m = sqrt(1.0 - ab), rsq = sqrt(ab), sqn = sqrt(ab_next), sq1mn = sqrt(1.0 - ab_next);
    const unsigned g = (unsigned)((n + 255) / 256);
    if (dtype == 0)
        ddim_update_kernel<double><<<g, 256, 0, (cudaStream_t)stream>>>((double*)x, (const double*)eps, n, sq1m, rsq,
                                                                         sqn, sq1mn, has_next, clip_lo, clip_hi,
                                                                         (double*)x0_out);
    else
        ddim_update_kernel<float><<<g, 256, 0, (cudaStream_t)stream>>>(
            (float*)x, (const float*)eps, n, (float)sq1m, (float)rsq, (float)sqn, (float)sq1mn, has_next,
            (float)clip_lo, (float)clip_hi, (float*)x0_out);
    PS_CHECK_LAUNCH();
    return PS_OK;
}
extern "C" int ps_ref_ddim_update(double* x, const double* eps, int n, double ab, double ab_next, int has_next,
                                  double clip_lo, double clip_hi, double* x0_out, void* stream) {
    return ps_ref_ddim_update_dt(0, x, eps, n, ab, ab_next, has_next, clip_lo, clip_hi, x0_out, stream);
}

// ---------------------------------------------------------------------------
// small elementwise helpers of the ref sampler (fp64)
// ---------------------------------------------------------------------------
namespace ps {
namespace ref {
// sinusoid of a 1-based step (src/diffusion.py:228-234): freq_i = exp(-ln(1e4) i / max(half-1, 1))
// (the angle in float64 for both types, rounded once: the features match to the last bit of F)
template <typename F>
__global__ void sinusoid_kernel(double k, int half, F* __restrict__ out) {
    const int i = threadIdx.x;
    if (i >= half) return;
    const double freq = exp(-log(10000.0) * (double)i / (double)(half > 1 ? half - 1 : 1));
    const double ang = k * freq;
    out[i] = (F)sin(ang);
    out[half + i] = (F)cos(ang);
}
template <typename F>
__global__ void div_kernel(const F* __restrict__ x, int n, F d, F* __restrict__ y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = x[i] / d;
}
// traj = lo + x0 * (hi - lo); row 0 := q0  (src/diffusion.py:559-569, arm.py:200-201)
template <typename F>
__global__ void denorm_pin_kernel(const F* __restrict__ x0, int B, int T, int D, const F* __restrict__ lo,
                                  const F* __restrict__ hi, const F* __restrict__ q0, F* __restrict__ traj) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B * T * D) return;
    const int d = i % D, t = (i / D) % T;
    traj[i] = t == 0 ? q0[d] : lo[d] + x0[i] * (hi[d] - lo[d]);
}
// select_best (src/pipeline.py:160-165) over fp64 costs, one thread per problem
__global__ void select_f64_kernel(const double* __restrict__ cost, const uint8_t* __restrict__ ok, int P, int S,
                                  int* __restrict__ best) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    bool any = false;
    for (int s = 0; s < S; ++s) any |= ok[p * S + s] != 0;
    int bi = -1;
    double bc = 0;
    for (int s = 0; s < S; ++s) {
        if (any && !ok[p * S + s]) continue;
        const double c = cost[p * S + s];
        if (bi < 0 || c < bc) {
            bi = s;
            bc = c;
        }
    }
    best[p] = bi;
}
}  // namespace ref
}  // namespace ps

extern "C" int ps_ref_sinusoid_dt(int dtype, double k, int half, void* out, void* stream) {
    if (half < 1 || half > 1024 || (dtype != 0 && dtype != 1)) return PS_FAIL(PS_ERR_SHAPE);
    if (dtype == 0) sinusoid_kernel<double><<<1, half, 0, (cudaStream_t)stream>>>(k, half, (double*)out);
    else sinusoid_kernel<float><<<1, half, 0, (cudaStream_t)stream>>>(k, half, (float*)out);
    PS_CHECK_LAUNCH();
    return PS_OK;
}
extern "C" int ps_ref_sinusoid(double k, int half, double* out, void* stream) {
    return ps_ref_sinusoid_dt(0, k, half, out, stream);
}
extern "C" int ps_ref_div_dt(int dtype, const void* x, int n, double d, void* y, void* stream) {
    if (n <= 0 || (dtype != 0 && dtype != 1)) return PS_FAIL(PS_ERR_SHAPE);
    const unsigned g = (unsigned)((n + 255) / 256);
    if (dtype == 0) div_kernel<double><<<g, 256, 0, (cudaStream_t)stream>>>((const double*)x, n, d, (double*)y);
    else div_kernel<float><<<g, 256, 0, (cudaStream_t)stream>>>((const float*)x, n, (float)d, (float*)y);
    PS_CHECK_LAUNCH();
    return PS_OK;
}
extern "C" int ps_ref_div(const double* x, int n, double d, double* y, void* stream) {
    return ps_ref_div_dt(0, x, n, d, y, stream);
}
extern "C" int ps_ref_denorm_pin_dt(int dtype, const void* x0, int B, int T, int D, const void* lo, const void* hi,
                                    const void* q0, void* traj, void* stream) {
    const int n = B * T * D;
    if (n <= 0 || (dtype != 0 && dtype != 1)) return PS_FAIL(PS_ERR_SHAPE);
    const unsigned g = (unsigned)((n + 255) / 256);
    if (dtype == 0)
        denorm_pin_kernel<double><<<g, 256, 0, (cudaStream_t)stream>>>((const double*)x0, B, T, D, (const double*)lo,
                                                                        (const double*)hi, (const double*)q0,
                                                                        (double*)traj);
    else
        denorm_pin_kernel<float><<<g, 256, 0, (cudaStream_t)stream>>>((const float*)x0, B, T, D, (const float*)lo,
                                                                       (const float*)hi, (const float*)q0,
                                                                       (float*)traj);
    PS_CHECK_LAUNCH();
    return PS_OK;
}
extern "C" int ps_ref_denorm_pin(const double* x0, int B, int T, int D, const double* lo, const double* hi,
                                 const double* q0, double* traj, void* stream) {
    return ps_ref_denorm_pin_dt(0, x0, B, T, D, lo, hi, q0, traj, stream);
}
extern "C" int ps_ref_select(const double* cost, const uint8_t* ok, int P, int S, int* best, void* stream) {
    if (P <= 0 || S <= 0) return PS_FAIL(PS_ERR_SHAPE);
    select_f64_kernel<<<(P + 63) / 64, 64, 0, (cudaStream_t)stream>>>(cost, ok, P, S, best);
    PS_CHECK_LAUNCH();
    return PS_OK;
}
