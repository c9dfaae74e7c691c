// BASELINE-profile refinement path: ESDF build, fused cost/gradient/fixed-step
// refinement with dense feasibility, and best-seed selection.
//
// Compiled with --fmad=false: all fused multiply-adds are explicit fmaf() in the
// canonical order of oracle/c/bl_oracle.c, so results are bit-identical to it.
//
// Layout: one warp per trajectory, lane l owns waypoints l*WPL .. l*WPL+WPL-1
// (T = 32*WPL).  Robot, weights and grid geometry travel in the kernel parameter
// block (__grid_constant__, constant bank broadcast); the trajectory state stays in
// registers for all iterations; the per-problem ESDF (128^3 fp32 = 8 MiB) is read
// through the read-only path with 8 scalar gathers per sphere lookup.
#include <algorithm>

#include <cstdlib>

#include <vector>

#include "common.cuh"

namespace ps {

constexpr int NJ = 7;
constexpr int MAX_SPH = 64;

struct BLParams {
    float dh[NJ][4];          // a, d, cos alpha, sin alpha
    float base[3];
    float sph[MAX_SPH][4];    // link-frame offset xyz, radius
    int link_start[NJ + 1];   // spheres of link k: [link_start[k], link_start[k+1])
    float w_coll, w_vel, w_acc, w_jerk, margin, eta;
    int nx, ny, nz;
    float ox, oy, oz, inv_h;
    int B, T, S, n_iters;
    int esdf_brick;           // ESDF layout: 0 C order, 1 4^3 bricks
    long long esdf_stride;
    const float* q_in;
    const float* esdf;
    float* q_out;
    float* cost;
    float* grad;
    uint8_t* feasible;
    uint8_t* clamped;
};

// World term of one configuration (canonical order, see bl_oracle.c:config_world).
template <bool WANT_GRAD, int PIPE = 1>
__device__ __forceinline__ void config_world(const BLParams& P, const Grid& g, const float (&q)[NJ],
                                             float& wc, float (&gq)[NJ], float& mc, bool& cl_any) {
    f3 X{1.f, 0.f, 0.f}, Y{0.f, 1.f, 0.f}, Z{0.f, 0.f, 1.f};
    f3 o{P.base[0], P.base[1], P.base[2]};
    f3 tz[NJ], tm[NJ];
    wc = 0.f;
    mc = __int_as_float(0x7f800000);
    cl_any = false;
    const float m2w = -2.0f * P.w_coll;
#pragma unroll
    for (int j = 0; j < NJ; ++j) gq[j] = 0.f;
#pragma unroll
    for (int k = 0; k < NJ; ++k) {
        tz[k] = Z;
        tm[k] = c_cross(o, Z);
        float sn, cs;
        c_sincos(q[k], sn, cs);
        const float a = P.dh[k][0], dd = P.dh[k][1], ca = P.dh[k][2], sa = P.dh[k][3];
        const float ac = a * cs, as = a * sn;
        o.x = fmaf(ac, X.x, fmaf(as, Y.x, fmaf(dd, Z.x, o.x)));
        o.y = fmaf(ac, X.y, fmaf(as, Y.y, fmaf(dd, Z.y, o.y)));
        o.z = fmaf(ac, X.z, fmaf(as, Y.z, fmaf(dd, Z.z, o.z)));
        f3 X1{fmaf(cs, X.x, sn * Y.x), fmaf(cs, X.y, sn * Y.y), fmaf(cs, X.z, sn * Y.z)};
        f3 Y1{fmaf(cs, Y.x, -(sn * X.x)), fmaf(cs, Y.y, -(sn * X.y)), fmaf(cs, Y.z, -(sn * X.z))};
        f3 Y2{fmaf(ca, Y1.x, sa * Z.x), fmaf(ca, Y1.y, sa * Z.y), fmaf(ca, Y1.z, sa * Z.z)};
        f3 Z2{fmaf(ca, Z.x, -(sa * Y1.x)), fmaf(ca, Z.y, -(sa * Y1.y)), fmaf(ca, Z.z, -(sa * Y1.z))};
        X = X1;
        Y = Y2;
        Z = Z2;
        f3 S1{0.f, 0.f, 0.f}, S2{0.f, 0.f, 0.f};
        const int s_end = P.link_start[k + 1];
        auto sphere_pos = [&](int s) {
            const float lx = P.sph[s][0], ly = P.sph[s][1], lz = P.sph[s][2];
            return f3{fmaf(X.x, lx, fmaf(Y.x, ly, fmaf(Z.x, lz, o.x))),
                      fmaf(X.y, lx, fmaf(Y.y, ly, fmaf(Z.y, lz, o.y))),
                      fmaf(X.z, lx, fmaf(Y.z, ly, fmaf(Z.z, lz, o.z)))};
        };
        auto accumulate = [&](int s, const f3& p, const TriCell& cell) {
            const float r = P.sph[s][3];
            f3 gr;
            const float dv = tri_eval(g, cell, gr);
            cl_any |= cell.clamped;
            mc = fminf(mc, dv - r);
            const float hinge = (r + P.margin) - dv;
            if (hinge > 0.f) {
                wc = fmaf(P.w_coll * hinge, hinge, wc);
                if (WANT_GRAD) {
                    const float coef = m2w * hinge;
                    f3 gp{coef * gr.x, coef * gr.y, coef * gr.z};
                    f3 cr = c_cross(p, gp);
                    S1.x = S1.x + cr.x; S1.y = S1.y + cr.y; S1.z = S1.z + cr.z;
                    S2.x = S2.x + gp.x; S2.y = S2.y + gp.y; S2.z = S2.z + gp.z;
                }
            }
        };
        // PIPE spheres per step: all their cells' corner loads are issued before any is
        // evaluated; the accumulation order stays sequential (bit-identical to the oracle)
        int s = P.link_start[k];
        if (PIPE >= 4)
        for (; s + 3 < s_end; s += 4) {
            f3 pp[4];
            TriCell cc[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                pp[u] = sphere_pos(s + u);
                tri_gather(g, pp[u], cc[u]);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) accumulate(s + u, pp[u], cc[u]);
        }
        if (PIPE >= 2)
        for (; s + 1 < s_end; s += 2) {
            const f3 pa = sphere_pos(s), pb = sphere_pos(s + 1);
            TriCell ca, cb;
            tri_gather(g, pa, ca);
            tri_gather(g, pb, cb);
            accumulate(s, pa, ca);
            accumulate(s + 1, pb, cb);
        }
        for (; s < s_end; ++s) {
            const f3 pa = sphere_pos(s);
            TriCell ca;
            tri_gather(g, pa, ca);
            accumulate(s, pa, ca);
        }
        if (WANT_GRAD) {
#pragma unroll
            for (int j = 0; j <= k; ++j) {
                float t = tz[j].x * S1.x;
                t = fmaf(tz[j].y, S1.y, t);
                t = fmaf(tz[j].z, S1.z, t);
                t = fmaf(tm[j].x, S2.x, t);
                t = fmaf(tm[j].y, S2.y, t);
                t = fmaf(tm[j].z, S2.z, t);
                gq[j] = gq[j] + t;
            }
        }
    }
}

// 3-term stencil of D (numpy.gradient, planseed/trajopt.py:64-73) or D^T across the
// warp's waypoints.  Missing neighbours are substituted by y_t (as the oracle does).
template <int WPL, bool TRANSPOSE>
__device__ __forceinline__ void stencil(const float (&y)[WPL], float (&out)[WPL], int lane, int T) {
    const float up = __shfl_up_sync(PS_FULL, y[WPL - 1], 1);
    const float dn = __shfl_down_sync(PS_FULL, y[0], 1);
#pragma unroll
    for (int w = 0; w < WPL; ++w) {
        const int t = lane * WPL + w;
        float ym = (w > 0) ? y[w > 0 ? w - 1 : 0] : (t == 0 ? y[w] : up);
        float yp = (w < WPL - 1) ? y[w < WPL - 1 ? w + 1 : w] : (t == T - 1 ? y[w] : dn);
        float cl, cs, cr;
        cs = (t == 0) ? -1.f : (t == T - 1 ? 1.f : 0.f);
        if (!TRANSPOSE) {
            cl = (t == 0) ? 0.f : (t == T - 1 ? -1.f : -0.5f);
            cr = (t == T - 1) ? 0.f : (t == 0 ? 1.f : 0.5f);
        } else {
            cl = (t == 0) ? 0.f : (t - 1 == 0 ? 1.f : 0.5f);
            cr = (t == T - 1) ? 0.f : (t + 1 == T - 1 ? -1.f : -0.5f);
        }
        float r = cs * y[w];
        r = fmaf(cl, ym, r);
        r = fmaf(cr, yp, r);
        out[w] = r;
    }
}

// Smoothness cost per waypoint and (optionally) gradient, see bl_oracle.c:smooth_terms.
template <int WPL, bool WANT_GRAD>
__device__ __forceinline__ void smooth_terms(const BLParams& P, const float (&q)[WPL][NJ], int lane,
                                             float (&sm)[WPL], float (&gs)[WPL][NJ]) {
#pragma unroll
    for (int w = 0; w < WPL; ++w) sm[w] = 0.f;
#pragma unroll
    for (int k = 0; k < NJ; ++k) {
        float y[WPL], v[WPL], a[WPL], jk[WPL];
#pragma unroll
        for (int w = 0; w < WPL; ++w) y[w] = q[w][k];
        stencil<WPL, false>(y, v, lane, P.T);
        stencil<WPL, false>(v, a, lane, P.T);
        stencil<WPL, false>(a, jk, lane, P.T);
#pragma unroll
        for (int w = 0; w < WPL; ++w) {
            float s = sm[w];
            s = fmaf(P.w_vel, v[w] * v[w], s);
            s = fmaf(P.w_acc, a[w] * a[w], s);
            s = fmaf(P.w_jerk, jk[w] * jk[w], s);
            sm[w] = s;
        }
        if (WANT_GRAD) {
            float z[WPL], zz[WPL], tmp[WPL];
#pragma unroll
            for (int w = 0; w < WPL; ++w) z[w] = P.w_jerk * jk[w];
            stencil<WPL, true>(z, tmp, lane, P.T);
#pragma unroll
            for (int w = 0; w < WPL; ++w) zz[w] = fmaf(P.w_acc, a[w], tmp[w]);
            stencil<WPL, true>(zz, tmp, lane, P.T);
#pragma unroll
            for (int w = 0; w < WPL; ++w) z[w] = fmaf(P.w_vel, v[w], tmp[w]);
            stencil<WPL, true>(z, tmp, lane, P.T);
#pragma unroll
            for (int w = 0; w < WPL; ++w) gs[w][k] = tmp[w];
        }
    }
}

__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = fminf(v, __shfl_xor_sync(PS_FULL, v, off));
    return v;
}

// MODE 0: refine (n_iters steps + final cost/flags).  MODE 1: cost + gradient only.
// LB: block-size bound -- 512 for throughput (one problem's 16 trajectories per block share
// the L1), 64 for small batches (up to 255 registers: the two-sphere gathers stay in flight)
template <int WPL, int MODE, int LB = 512, int PIPE = 1>
__global__ void __launch_bounds__(LB) bl_refine_kernel(const __grid_constant__ BLParams P) {
    const int lane = threadIdx.x & 31;
    const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (b >= P.B) return;  // whole warp exits together
    Grid g;
    g.v = P.esdf + (size_t)(b / P.S) * (size_t)P.esdf_stride;
    g.nx = P.nx; g.ny = P.ny; g.nz = P.nz;
    g.ox = P.ox; g.oy = P.oy; g.oz = P.oz; g.inv_h = P.inv_h;
    g.brick = P.esdf_brick;

    float q[WPL][NJ];
    const float* qb = P.q_in + (size_t)b * P.T * NJ;
#pragma unroll
    for (int w = 0; w < WPL; ++w)
#pragma unroll
        for (int k = 0; k < NJ; ++k) q[w][k] = qb[(lane * WPL + w) * NJ + k];

    float sm[WPL], gs[WPL][NJ];
    if constexpr (MODE == 1) {
        float ct[WPL];
        bool cl_lane = false;
        smooth_terms<WPL, true>(P, q, lane, sm, gs);
#pragma unroll
        for (int w = 0; w < WPL; ++w) {
            float wc, mc, gq[NJ];
            bool cl;
            config_world<true, PIPE>(P, g, q[w], wc, gq, mc, cl);
            cl_lane |= cl;
            ct[w] = wc + sm[w];
            const int t = lane * WPL + w;
            float* gout = P.grad + ((size_t)b * P.T + t) * NJ;
#pragma unroll
            for (int k = 0; k < NJ; ++k) gout[k] = (t == 0) ? 0.f : fmaf(2.0f, gs[w][k], gq[k]);
        }
        float c = ct[0];
#pragma unroll
        for (int w = 1; w < WPL; ++w) c = c + ct[w];
        c = warp_sum_butterfly(c);
        const bool cl_any = __any_sync(PS_FULL, cl_lane);
        if (lane == 0) {
            P.cost[b] = c;
            P.clamped[b] = cl_any ? 1 : 0;
        }
        return;
    }

    for (int it = 0; it < P.n_iters; ++it) {
        float gw[WPL][NJ];
#pragma unroll
        for (int w = 0; w < WPL; ++w) {
            float wc, mc;
            bool cl;
            config_world<true, PIPE>(P, g, q[w], wc, gw[w], mc, cl);
        }
        smooth_terms<WPL, true>(P, q, lane, sm, gs);
#pragma unroll
        for (int w = 0; w < WPL; ++w) {
            const int t = lane * WPL + w;
            if (t != 0) {
#pragma unroll
                for (int k = 0; k < NJ; ++k) q[w][k] = fmaf(-P.eta, fmaf(2.0f, gs[w][k], gw[w][k]), q[w][k]);
            }
        }
    }

    // final cost, clearance and clamped flag at the waypoints
    smooth_terms<WPL, false>(P, q, lane, sm, gs);
    float ct[WPL];
    float mc_lane = __int_as_float(0x7f800000);
    bool cl_lane = false;
#pragma unroll
    for (int w = 0; w < WPL; ++w) {
        float wc, mc, gq[NJ];
        bool cl;
        config_world<false, PIPE>(P, g, q[w], wc, gq, mc, cl);
        ct[w] = wc + sm[w];
        mc_lane = fminf(mc_lane, mc);
        cl_lane |= cl;
    }
    // dense check: 4 interpolants per segment (planseed/pipeline.py:139-157)
    float qn[NJ];
#pragma unroll
    for (int k = 0; k < NJ; ++k) qn[k] = __shfl_down_sync(PS_FULL, q[0][k], 1);
#pragma unroll
    for (int w = 0; w < WPL; ++w) {
        const int t = lane * WPL + w;
        if (t + 1 < P.T) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float f = (float)(i + 1) / 5.0f;
                float qi[NJ], wc, mc, gq[NJ];
                bool cl;
#pragma unroll
                for (int k = 0; k < NJ; ++k) {
                    const float q1 = (w + 1 < WPL) ? q[w + 1 < WPL ? w + 1 : w][k] : qn[k];
                    qi[k] = fmaf(f, q1 - q[w][k], q[w][k]);
                }
                config_world<false, PIPE>(P, g, qi, wc, gq, mc, cl);
                mc_lane = fminf(mc_lane, mc);
                cl_lane |= cl;
            }
        }
    }
    float c = ct[0];
#pragma unroll
    for (int w = 1; w < WPL; ++w) c = c + ct[w];
    c = warp_sum_butterfly(c);
    const float mc_all = warp_min(mc_lane);
    const bool cl_any = __any_sync(PS_FULL, cl_lane);
    float* qo = P.q_out + (size_t)b * P.T * NJ;
#pragma unroll
    for (int w = 0; w < WPL; ++w)
#pragma unroll
        for (int k = 0; k < NJ; ++k) qo[(lane * WPL + w) * NJ + k] = q[w][k];
    if (lane == 0) {
        P.cost[b] = c;
        P.feasible[b] = (mc_all > 0.f) ? 1 : 0;
        P.clamped[b] = cl_any ? 1 : 0;
    }
}

// ---------------------------------------------------------------------------
// Cost-guided sampling's guide step (guided_ddim_sample, planseed/diffusion.py:572-628) for the BL
// cost: per trajectory (one warp), n_grad descent steps on the normalised x0_hat, each from step
// alpha with <= max_halvings halvings until the cost of the denormalised candidate decreases.
// Seeds are independent (their costs never mix), so the whole guide step is one launch.  The
// evaluation order is orc_bl_guide's (oracle/c/bl_oracle.c): bit-identical results.
// ---------------------------------------------------------------------------
struct BLGuideArgs {
    float* x;                 // (B, T, 7) normalised x0_hat, in place
    float lo[NJ], span[NJ];   // denormalise: q = lo + x * span
    int n_grad, max_halvings;
    float alpha;
    uint8_t* clamped;         // (B,) some evaluation left the ESDF extent
};

template <int WPL, bool GRAD>
__device__ __forceinline__ float traj_cost_dev(const BLParams& P, const Grid& g, const float (&q)[WPL][NJ], int lane,
                                               float (&grad)[WPL][NJ], bool& cl_any) {
    float sm[WPL], gs[WPL][NJ], ct[WPL];
    smooth_terms<WPL, GRAD>(P, q, lane, sm, gs);
    bool cl_lane = false;
#pragma unroll
    for (int w = 0; w < WPL; ++w) {
        float wc, mc, gq[NJ];
        bool cl;
        config_world<GRAD, 1>(P, g, q[w], wc, gq, mc, cl);
        cl_lane |= cl;
        ct[w] = wc + sm[w];
        if (GRAD) {
            const int t = lane * WPL + w;
#pragma unroll
            for (int k = 0; k < NJ; ++k) grad[w][k] = (t == 0) ? 0.f : fmaf(2.0f, gs[w][k], gq[k]);
        }
    }
    float c = ct[0];
#pragma unroll
    for (int w = 1; w < WPL; ++w) c = c + ct[w];
    cl_any = __any_sync(PS_FULL, cl_lane);
    return warp_sum_butterfly(c);
}

template <int WPL>
__global__ void __launch_bounds__(256) bl_guide_kernel(const __grid_constant__ BLParams P,
                                                        const __grid_constant__ BLGuideArgs A) {
    const int lane = threadIdx.x & 31;
    const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (b >= P.B) return;   // whole warp
    Grid g;
    g.v = P.esdf + (size_t)(b / P.S) * (size_t)P.esdf_stride;
    g.nx = P.nx; g.ny = P.ny; g.nz = P.nz;
    g.ox = P.ox; g.oy = P.oy; g.oz = P.oz; g.inv_h = P.inv_h;
    g.brick = P.esdf_brick;
    float x[WPL][NJ], q[WPL][NJ], gr[WPL][NJ];
    float* xb = A.x + (size_t)b * P.T * NJ;
#pragma unroll
    for (int w = 0; w < WPL; ++w)
#pragma unroll
        for (int k = 0; k < NJ; ++k) x[w][k] = xb[(lane * WPL + w) * NJ + k];
    bool cl_any = false;
    for (int it = 0; it < A.n_grad; ++it) {
#pragma unroll
        for (int w = 0; w < WPL; ++w)
#pragma unroll
            for (int k = 0; k < NJ; ++k) q[w][k] = A.lo[k] + x[w][k] * A.span[k];
        bool cl;
        const float c = traj_cost_dev<WPL, true>(P, g, q, lane, gr, cl);
        cl_any |= cl;
#pragma unroll
        for (int w = 0; w < WPL; ++w)
#pragma unroll
            for (int k = 0; k < NJ; ++k) gr[w][k] = gr[w][k] * A.span[k];
        float step = A.alpha;
        for (int hv = 0; hv < A.max_halvings; ++hv) {
            float cand[WPL][NJ];
#pragma unroll
            for (int w = 0; w < WPL; ++w)
#pragma unroll
                for (int k = 0; k < NJ; ++k) {
                    cand[w][k] = x[w][k] - step * gr[w][k];
                    q[w][k] = A.lo[k] + cand[w][k] * A.span[k];
                }
            float dummy[WPL][NJ];
            const float cn = traj_cost_dev<WPL, false>(P, g, q, lane, dummy, cl);
            cl_any |= cl;
            if (cn < c) {   // warp-uniform: both costs are warp-reduced
#pragma unroll
                for (int w = 0; w < WPL; ++w)
#pragma unroll
                    for (int k = 0; k < NJ; ++k) x[w][k] = cand[w][k];
                break;
            }
            step = step * 0.5f;
        }
    }
#pragma unroll
    for (int w = 0; w < WPL; ++w)
#pragma unroll
        for (int k = 0; k < NJ; ++k) xb[(lane * WPL + w) * NJ + k] = x[w][k];
    if (lane == 0) A.clamped[b] = cl_any ? 1 : 0;
}

// ---------------------------------------------------------------------------
// Ground-truth evaluation (trajopt.metrics / retime / traj_min_clearance, planseed/trajopt.py:
// 209-272, _kernels.py:144-162) against the problem's analytic boxes: one warp per trajectory,
// lane = waypoint(s).  Clearance = min over waypoints + interp interpolants per segment of
// min over spheres of (box SDF at the centre - radius), capped; end-pose errors of the frame after
// joint 7; uniform retiming from the D / D^2 / D^3 stencils and the per-joint limits.
// ---------------------------------------------------------------------------
struct BLMetricArgs {
    const float* traj;        // (B, T, 7)
    const float* boxes;       // (P, n_boxes, 6)
    const float* goal;        // (P, 7): xyz relative to the base, quaternion (w, x, y, z)
    int n_boxes, interp;
    float cap, vel, acc, jerk, delta_t, delta_r_deg;
    float* clearance;         // (B,)
    float* terr;
    float* aerr_deg;
    float* motion_time;
    float* max_jerk;
    uint8_t* success;
    uint8_t* collision_free;
};

// FK of one configuration; calls f(link k, X, Y, Z, o) after each joint (frame k+1)
template <typename F>
__device__ __forceinline__ void fk_frames(const BLParams& P, const float (&q)[NJ], F&& f) {
    f3 X{1.f, 0.f, 0.f}, Y{0.f, 1.f, 0.f}, Z{0.f, 0.f, 1.f};
    f3 o{P.base[0], P.base[1], P.base[2]};
#pragma unroll
    for (int k = 0; k < NJ; ++k) {
        float sn, cs;
        c_sincos(q[k], sn, cs);
        const float a = P.dh[k][0], dd = P.dh[k][1], ca = P.dh[k][2], sa = P.dh[k][3];
        const float ac = a * cs, as = a * sn;
        o.x = fmaf(ac, X.x, fmaf(as, Y.x, fmaf(dd, Z.x, o.x)));
        o.y = fmaf(ac, X.y, fmaf(as, Y.y, fmaf(dd, Z.y, o.y)));
        o.z = fmaf(ac, X.z, fmaf(as, Y.z, fmaf(dd, Z.z, o.z)));
        f3 X1{fmaf(cs, X.x, sn * Y.x), fmaf(cs, X.y, sn * Y.y), fmaf(cs, X.z, sn * Y.z)};
        f3 Y1{fmaf(cs, Y.x, -(sn * X.x)), fmaf(cs, Y.y, -(sn * X.y)), fmaf(cs, Y.z, -(sn * X.z))};
        f3 Y2{fmaf(ca, Y1.x, sa * Z.x), fmaf(ca, Y1.y, sa * Z.y), fmaf(ca, Y1.z, sa * Z.z)};
        f3 Z2{fmaf(ca, Z.x, -(sa * Y1.x)), fmaf(ca, Z.y, -(sa * Y1.y)), fmaf(ca, Z.z, -(sa * Y1.z))};
        X = X1;
        Y = Y2;
        Z = Z2;
        f(k, X, Y, Z, o);
    }
}

__device__ __forceinline__ float config_clearance3(const BLParams& P, const float (&q)[NJ], const float* bx, int nb,
                                                   float cap) {
    float best = cap;
    fk_frames(P, q, [&](int k, const f3& X, const f3& Y, const f3& Z, const f3& o) {
        for (int s = P.link_start[k]; s < P.link_start[k + 1]; ++s) {
            const float lx = P.sph[s][0], ly = P.sph[s][1], lz = P.sph[s][2];
            const float px = fmaf(X.x, lx, fmaf(Y.x, ly, fmaf(Z.x, lz, o.x)));
            const float py = fmaf(X.y, lx, fmaf(Y.y, ly, fmaf(Z.y, lz, o.y)));
            const float pz = fmaf(X.z, lx, fmaf(Y.z, ly, fmaf(Z.z, lz, o.z)));
            float d = cap;
            for (int b = 0; b < nb; ++b) {
                const float* c = bx + 6 * b;   // centre, half extent
                const float qx = fabsf(px - c[0]) - c[3], qy = fabsf(py - c[1]) - c[4], qz = fabsf(pz - c[2]) - c[5];
                const float ax = fmaxf(qx, 0.f), ay = fmaxf(qy, 0.f), az = fmaxf(qz, 0.f);
                d = fminf(d, sqrtf(fmaf(ax, ax, fmaf(ay, ay, az * az))) + fminf(fmaxf(qx, fmaxf(qy, qz)), 0.f));
            }
            best = fminf(best, d - P.sph[s][3]);
        }
    });
    return best;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = fmaxf(v, __shfl_xor_sync(PS_FULL, v, off));
    return v;
}

template <int WPL>
__global__ void __launch_bounds__(256) bl_metrics_kernel(const __grid_constant__ BLParams P,
                                                          const __grid_constant__ BLMetricArgs M) {
    __shared__ float s_box[8][64 * 6];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (b >= P.B) return;   // whole warp
    const int p = b / P.S;
    float* bx = s_box[wib];
    for (int i = lane; i < M.n_boxes * 3; i += 32) {
        const int k = i / 3, a = i % 3;
        const float lo = M.boxes[((size_t)p * M.n_boxes + k) * 6 + a], hi = M.boxes[((size_t)p * M.n_boxes + k) * 6 + 3 + a];
        bx[6 * k + a] = 0.5f * (lo + hi);
        bx[6 * k + 3 + a] = 0.5f * (hi - lo);
    }
    __syncwarp();
    float q[WPL][NJ];
    const float* qb = M.traj + (size_t)b * P.T * NJ;
#pragma unroll
    for (int w = 0; w < WPL; ++w)
#pragma unroll
        for (int k = 0; k < NJ; ++k) q[w][k] = qb[(lane * WPL + w) * NJ + k];
    // clearance at the waypoints and the interpolants toward the next waypoint
    float qn[NJ];
#pragma unroll
    for (int k = 0; k < NJ; ++k) qn[k] = __shfl_down_sync(PS_FULL, q[0][k], 1);
    float clr = M.cap;
#pragma unroll
    for (int w = 0; w < WPL; ++w) {
        clr = fminf(clr, config_clearance3(P, q[w], bx, M.n_boxes, M.cap));
        const int t = lane * WPL + w;
        if (t + 1 < P.T) {
            for (int i = 0; i < M.interp; ++i) {
                const float f = (float)(i + 1) / (float)(M.interp + 1);
                float qi[NJ];
#pragma unroll
                for (int k = 0; k < NJ; ++k) {
                    const float q1 = (w + 1 < WPL) ? q[w + 1 < WPL ? w + 1 : w][k] : qn[k];
                    qi[k] = fmaf(f, q1 - q[w][k], q[w][k]);
                }
                clr = fminf(clr, config_clearance3(P, qi, bx, M.n_boxes, M.cap));
            }
        }
    }
    clr = warp_min(clr);
    // retiming: per-joint max |D q|, |D^2 q|, |D^3 q| over the trajectory
    float rv = 0.f, ra = 0.f, rj = 0.f, jmax = 0.f;
#pragma unroll
    for (int k = 0; k < NJ; ++k) {
        float y[WPL], v[WPL], a[WPL], jk[WPL];
#pragma unroll
        for (int w = 0; w < WPL; ++w) y[w] = q[w][k];
        stencil<WPL, false>(y, v, lane, P.T);
        stencil<WPL, false>(v, a, lane, P.T);
        stencil<WPL, false>(a, jk, lane, P.T);
        float mv = 0.f, ma = 0.f, mj = 0.f;
#pragma unroll
        for (int w = 0; w < WPL; ++w) {
            mv = fmaxf(mv, fabsf(v[w]));
            ma = fmaxf(ma, fabsf(a[w]));
            mj = fmaxf(mj, fabsf(jk[w]));
        }
        mv = warp_max(mv);
        ma = warp_max(ma);
        mj = warp_max(mj);
        rv = fmaxf(rv, mv / M.vel);
        ra = fmaxf(ra, ma / M.acc);
        rj = fmaxf(rj, mj / M.jerk);
        jmax = fmaxf(jmax, mj);
    }
    const float dt = fmaxf(rv, fmaxf(sqrtf(ra), cbrtf(rj)));
    const float mt = dt * (float)(P.T - 1);
    // end pose: the lane holding the last waypoint
    if (lane == (P.T - 1) / WPL) {
        float ql[NJ];
#pragma unroll
        for (int k = 0; k < NJ; ++k) ql[k] = q[WPL - 1][k];
        f3 E[3], oe{0.f, 0.f, 0.f};
        fk_frames(P, ql, [&](int k, const f3& X, const f3& Y, const f3& Z, const f3& o) {
            if (k == NJ - 1) {
                E[0] = X; E[1] = Y; E[2] = Z; oe = o;
            }
        });
        const float* g = M.goal + (size_t)p * 7;
        const float dx = (oe.x - P.base[0]) - g[0], dy = (oe.y - P.base[1]) - g[1], dz = (oe.z - P.base[2]) - g[2];
        const float terr = sqrtf(dx * dx + dy * dy + dz * dz);
        const float w = g[3], x = g[4], y = g[5], z = g[6];
        const f3 G[3] = {{1.f - 2.f * (y * y + z * z), 2.f * (x * y + z * w), 2.f * (x * z - y * w)},
                         {2.f * (x * y - z * w), 1.f - 2.f * (x * x + z * z), 2.f * (y * z + x * w)},
                         {2.f * (x * z + y * w), 2.f * (y * z - x * w), 1.f - 2.f * (x * x + y * y)}};
        auto dot = [](const f3& u, const f3& v) { return u.x * v.x + u.y * v.y + u.z * v.z; };
        const float tr = dot(G[0], E[0]) + dot(G[1], E[1]) + dot(G[2], E[2]);
        const float v0 = dot(G[2], E[1]) - dot(G[1], E[2]), v1 = dot(G[0], E[2]) - dot(G[2], E[0]),
                    v2 = dot(G[1], E[0]) - dot(G[0], E[1]);
        const float aerr = atan2f(sqrtf(v0 * v0 + v1 * v1 + v2 * v2), tr - 1.f) * 57.29577951308232f;
        const bool free_ = clr > 0.f;
        M.clearance[b] = clr;
        M.terr[b] = terr;
        M.aerr_deg[b] = aerr;
        M.motion_time[b] = mt;
        M.max_jerk[b] = mt > 0.f ? jmax / (dt * dt * dt) : 0.f;
        M.collision_free[b] = free_ ? 1 : 0;
        M.success[b] = (free_ && terr <= M.delta_t && aerr <= M.delta_r_deg) ? 1 : 0;
    }
}

// ---------------------------------------------------------------------------
// ESDF build: 4 consecutive z nodes per thread, float4 store (nz % 4 == 0).
// ---------------------------------------------------------------------------
constexpr int MAX_BOXES = 64;

template <int VEC>
__global__ void __launch_bounds__(256) esdf_boxes_kernel(const float* __restrict__ boxes, int n_boxes,
                                                         int nx, int ny, int nz, float ox, float oy,
                                                         float oz, float h, float cap,
                                                         float* __restrict__ out) {
    __shared__ float bc[MAX_BOXES][3], bh[MAX_BOXES][3];
    const int p = blockIdx.y;
    const float* bx = boxes + (size_t)p * n_boxes * 6;
    for (int i = threadIdx.x; i < n_boxes * 3; i += blockDim.x) {
        const int b = i / 3, a = i % 3;
        const float lo = bx[b * 6 + a], hi = bx[b * 6 + 3 + a];
        bc[b][a] = 0.5f * (lo + hi);
        bh[b][a] = 0.5f * (hi - lo);
    }
    __syncthreads();
    const long long n_nodes = (long long)nx * ny * nz;
    const long long first = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * VEC;
    if (first >= n_nodes) return;
    const int k0 = (int)(first % nz);
    const long long ij = first / nz;
    const int j = (int)(ij % ny), i = (int)(ij / ny);
    const float px = fmaf((float)i, h, ox), py = fmaf((float)j, h, oy);
    float res[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
        const float pz = fmaf((float)(k0 + v), h, oz);
        float best = cap;
        for (int b = 0; b < n_boxes; ++b) {
            const float qx = fabsf(px - bc[b][0]) - bh[b][0];
            const float qy = fabsf(py - bc[b][1]) - bh[b][1];
            const float qz = fabsf(pz - bc[b][2]) - bh[b][2];
            const float ax = fmaxf(qx, 0.f), ay = fmaxf(qy, 0.f), az = fmaxf(qz, 0.f);
            const float outside = sqrtf(fmaf(ax, ax, fmaf(ay, ay, az * az)));
            const float inside = fminf(fmaxf(qx, fmaxf(qy, qz)), 0.f);
            best = fminf(best, outside + inside);
        }
        res[v] = best;
    }
    float* o = out + (size_t)p * (size_t)n_nodes + first;
    if (VEC == 4) {
        *reinterpret_cast<float4*>(o) = make_float4(res[0], res[1], res[2], res[VEC > 3 ? 3 : 0]);
    } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) o[v] = res[v];
    }
}

// ---------------------------------------------------------------------------
// ESDF build with exact box culling: one warp per (x, y) column, lanes along z (4 nodes
// each).  For a column, lb_b = fmaf(ax, ax, ay*ay) (the squared-distance FMA chain without
// the z term) bounds every node's squared distance term from below (monotone rounding).
// Boxes are visited in ascending lb order and the walk stops once lb > 0 && lb >= every
// node's running min of the squared term, which cannot change any minimum; the sqrtf is
// taken once per node.  Results are bit-identical to the all-boxes loop (see below).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) esdf_cull_kernel(const float* __restrict__ boxes, int n_boxes, int nx, int ny,
                                                        int nz, float ox, float oy, float oz, float h, float cap,
                                                        float* __restrict__ out, int brick) {
    // per warp, the column's boxes sorted by their xy lower bound, with the column-constant
    // parts of the box distance (ax, ay, max(qx, qy)) precomputed
    __shared__ float s_lb[8][32], s_cz[8][32], s_hz[8][32], s_ax[8][32], s_ay[8][32], s_mq[8][32];
    __shared__ float bc[32][3], bh[32][3];
    const int p = blockIdx.y;
    const float* bx = boxes + (size_t)p * n_boxes * 6;
    for (int i = threadIdx.x; i < n_boxes * 3; i += blockDim.x) {
        const int b = i / 3, a = i % 3;
        const float lo = bx[b * 6 + a], hi = bx[b * 6 + 3 + a];
        bc[b][a] = 0.5f * (lo + hi);
        bh[b][a] = 0.5f * (hi - lo);
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long n_nodes = (long long)nx * ny * nz;
    const int n_col = nx * ny;
    for (int col = blockIdx.x * 8 + warp; col < n_col; col += gridDim.x * 8) {
        const int i = col / ny, j = col % ny;
        const float px = fmaf((float)i, h, ox), py = fmaf((float)j, h, oy);
        // column lower bound in squared form: every node's fmaf(ax,ax, fmaf(ay,ay, az*az)) is
        // >= fmaf(ax,ax, ay*ay) (monotone rounding), and sqrtf is monotone
        float lb = __int_as_float(0x7f800000);
        int id = lane;
        if (lane < n_boxes) {
            const float qx = fabsf(px - bc[lane][0]) - bh[lane][0];
            const float qy = fabsf(py - bc[lane][1]) - bh[lane][1];
            const float ax = fmaxf(qx, 0.f), ay = fmaxf(qy, 0.f);
            lb = fmaf(ax, ax, ay * ay);
        }
        // bitonic sort of (lb, id) across the warp, ascending
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
            for (int jj = k >> 1; jj > 0; jj >>= 1) {
                const float olb = __shfl_xor_sync(PS_FULL, lb, jj);
                const int oid = __shfl_xor_sync(PS_FULL, id, jj);
                const bool up = ((lane & k) == 0);
                const bool lower = (lane & jj) == 0;
                const bool o_less = (olb < lb) || (olb == lb && oid < id);
                const bool take = lower ? (up ? o_less : !o_less) : (up ? !o_less : o_less);
                if (take) {
                    lb = olb;
                    id = oid;
                }
            }
        }
        if (lane < n_boxes) {
            const float qx = fabsf(px - bc[id][0]) - bh[id][0];
            const float qy = fabsf(py - bc[id][1]) - bh[id][1];
            s_lb[warp][lane] = lb;
            s_cz[warp][lane] = bc[id][2];
            s_hz[warp][lane] = bh[id][2];
            s_ax[warp][lane] = fmaxf(qx, 0.f);
            s_ay[warp][lane] = fmaxf(qy, 0.f);
            s_mq[warp][lane] = fmaxf(qx, qy);   // fmaxf is exact: max(qx, qy, qz) in any order
        }
        __syncwarp();
        float* o = out + (size_t)p * (size_t)n_nodes + (size_t)col * nz;
        // Each lane owns 4 adjacent nodes (k = 4 lane + m).  Per box d_b = sqrtf(X_b) + min(max q, 0):
        // a box containing the node has X_b = 0 and d_b = max q < 0, any other box has
        // d_b = sqrtf(X_b).  So min_b d_b = min(sqrtf(min_b X_b), min of the negative max q),
        // bit-identical to the per-box sum (sqrtf is correctly rounded and monotone, x + 0 = x),
        // with one sqrtf per node.  The walk over the sorted boxes stops once the next box's
        // squared xy bound is positive and >= every node's min X.
        for (int k0 = 0; k0 < nz; k0 += 128) {
            float pz[4], mx[4], mi[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                pz[m] = fmaf((float)(k0 + 4 * lane + m), h, oz);   // 4 adjacent nodes: tight walk
                mx[m] = __int_as_float(0x7f800000);
                mi[m] = __int_as_float(0x7f800000);
            }
            // z-aware bound of the lane's 4 nodes: their z distance to the box is at least
            // |mid - cz| - hz - 1.5 h (minus slack for the rounding of the node coordinates)
            const float pmid = fmaf((float)(k0 + 4 * lane) + 1.5f, h, oz);
            const float zslack = fmaf(1.5f, h, 1e-5f);
            for (int e = 0; e < n_boxes; ++e) {
                const float l = s_lb[warp][e];
                const float bmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
                if (l > 0.f && l >= bmax) break;
                const float cz = s_cz[warp][e], hz = s_hz[warp][e];
                const float ax = s_ax[warp][e], ay = s_ay[warp][e], mq = s_mq[warp][e];
                const float azl = fmaxf(fabsf(pmid - cz) - hz - zslack, 0.f);
                const float lbz = fmaf(ax, ax, fmaf(ay, ay, azl * azl));
                if (lbz > 0.f && lbz >= bmax) continue;   // cannot lower any of the 4 minima
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const float qz = fabsf(pz[m] - cz) - hz;
                    const float az = fmaxf(qz, 0.f);
                    mx[m] = fminf(mx[m], fmaf(ax, ax, fmaf(ay, ay, az * az)));
                    mi[m] = fminf(mi[m], fmaxf(mq, qz));
                }
            }
            float res[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                res[m] = fminf(cap, sqrtf(mx[m]));
                if (mi[m] < 0.f) res[m] = fminf(res[m], mi[m]);
            }
            const int kk = k0 + 4 * lane;
            if (brick) {   // 4 nodes = one brick row (k..k+3, k % 4 == 0)
                if (kk < nz)
                    *reinterpret_cast<float4*>(out + (size_t)p * (size_t)n_nodes + esdf_brick_index(i, j, kk, ny, nz)) =
                        make_float4(res[0], res[1], res[2], res[3]);
            } else if (kk + 3 < nz && (nz & 3) == 0) {
                *reinterpret_cast<float4*>(o + kk) = make_float4(res[0], res[1], res[2], res[3]);
            } else {
#pragma unroll
                for (int m = 0; m < 4; ++m)
                    if (kk + m < nz) o[kk + m] = res[m];
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// ESDF build with 3-D tile culling: one warp per 8x8x8-node tile (2x2x2 bricks of 4^3).
// Lane b < n_boxes bounds box b's signed distance over the tile: L_b <= d_b(n) <= U_b for every
// node n (L_b: the box-to-tile-AABB distance, -inf when they overlap; U_b: the largest corner
// value -- a box's signed distance is convex, so its maximum over the tile is at a corner), both
// padded by a margin far above the fp32 rounding of the node expression.  With U* = min(cap,
// min_b U_b) >= every node's result, a box with L_b > U* cannot be any node's minimum and is
// skipped for the whole tile; typically 1-4 of 20 boxes survive.  The survivors are evaluated
// per node with the canonical expression, and min over a superset of the argmin boxes equals the
// min over all boxes, so results stay bit-identical to orc_esdf_build (see esdf_cull_kernel for
// the sqrtf / inside-term identity).  Lane l writes 4 rows of 4 k-adjacent nodes (float4, one
// brick row in either layout).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) esdf_tile_kernel(const float* __restrict__ boxes, int n_boxes, int P, int nx,
                                                        int ny, int nz, float ox, float oy, float oz, float h,
                                                        float cap, float* __restrict__ out, int brick) {
    const int lane = threadIdx.x & 31;
    const int tx = (nx + 7) >> 3, ty = (ny + 7) >> 3, tz = (nz + 7) >> 3;
    const long long tiles_per = (long long)tx * ty * tz, n_tiles = tiles_per * P;
    const long long n_nodes = (long long)nx * ny * nz;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    int cur_p = -1;
    float cx = 0.f, cy = 0.f, cz = 0.f, hx = 0.f, hy = 0.f, hz = 0.f;
    for (long long t = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < n_tiles; t += warps) {
        const int p = (int)(t / tiles_per);
        long long r = t - (long long)p * tiles_per;
        const int ti = (int)(r / ((long long)ty * tz));
        r -= (long long)ti * ty * tz;
        const int tj = (int)(r / tz), tk = (int)(r - (long long)tj * tz);
        if (p != cur_p) {   // box b (centre, half extent) in lane b, as the oracle computes them
            cur_p = p;
            if (lane < n_boxes) {
                const float* bx = boxes + ((size_t)p * n_boxes + lane) * 6;
                cx = 0.5f * (bx[0] + bx[3]); hx = 0.5f * (bx[3] - bx[0]);
                cy = 0.5f * (bx[1] + bx[4]); hy = 0.5f * (bx[4] - bx[1]);
                cz = 0.5f * (bx[2] + bx[5]); hz = 0.5f * (bx[5] - bx[2]);
            }
        }
        const int i0 = ti * 8, j0 = tj * 8, k0 = tk * 8;
        const int i1 = min(i0 + 8, nx) - 1, j1 = min(j0 + 8, ny) - 1, k1 = min(k0 + 8, nz) - 1;
        // tile AABB of the node positions
        const float xa = fmaf((float)i0, h, ox), xb = fmaf((float)i1, h, ox);
        const float ya = fmaf((float)j0, h, oy), yb = fmaf((float)j1, h, oy);
        const float za = fmaf((float)k0, h, oz), zb = fmaf((float)k1, h, oz);
        float L = __int_as_float(0x7f800000), U = __int_as_float(0x7f800000);
        if (lane < n_boxes) {
            const float gx = fmaxf(fmaxf((cx - hx) - xb, xa - (cx + hx)), 0.f);
            const float gy = fmaxf(fmaxf((cy - hy) - yb, ya - (cy + hy)), 0.f);
            const float gz = fmaxf(fmaxf((cz - hz) - zb, za - (cz + hz)), 0.f);
            const float gg = gx * gx + gy * gy + gz * gz;
            L = gg > 0.f ? sqrtf(gg) * (1.f - 1e-5f) - 1e-5f : -__int_as_float(0x7f800000);
            float u = -__int_as_float(0x7f800000);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const float qx = fabsf(((c & 1) ? xb : xa) - cx) - hx;
                const float qy = fabsf(((c & 2) ? yb : ya) - cy) - hy;
                const float qz = fabsf(((c & 4) ? zb : za) - cz) - hz;
                const float ax = fmaxf(qx, 0.f), ay = fmaxf(qy, 0.f), az = fmaxf(qz, 0.f);
                u = fmaxf(u, sqrtf(ax * ax + ay * ay + az * az) + fminf(fmaxf(qx, fmaxf(qy, qz)), 0.f));
            }
            U = u + 1e-5f * (1.f + fabsf(u));
        }
        float ustar = fminf(U, cap);
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) ustar = fminf(ustar, __shfl_xor_sync(PS_FULL, ustar, off));
        unsigned live = __ballot_sync(PS_FULL, lane < n_boxes && !(L > ustar));
        // this lane's 4 rows: (i0 + (lane >> 4) + 2m, j0 + ((lane >> 1) & 7), k0 + 4 (lane & 1))
        const int jj = j0 + ((lane >> 1) & 7), kk = k0 + 4 * (lane & 1);
        const float py = fmaf((float)jj, h, oy);
        float pz[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) pz[e] = fmaf((float)(kk + e), h, oz);
        float mx[4][4], mi[4][4];
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                mx[m][e] = __int_as_float(0x7f800000);
                mi[m][e] = __int_as_float(0x7f800000);
            }
        while (live) {
            const int b = __ffs(live) - 1;
            live &= live - 1;
            const float bcx = __shfl_sync(PS_FULL, cx, b), bhx = __shfl_sync(PS_FULL, hx, b);
            const float bcy = __shfl_sync(PS_FULL, cy, b), bhy = __shfl_sync(PS_FULL, hy, b);
            const float bcz = __shfl_sync(PS_FULL, cz, b), bhz = __shfl_sync(PS_FULL, hz, b);
            const float qy = fabsf(py - bcy) - bhy;
            const float ay = fmaxf(qy, 0.f);
            float qz[4], az2[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                qz[e] = fabsf(pz[e] - bcz) - bhz;
                const float az = fmaxf(qz[e], 0.f);
                az2[e] = fmaf(ay, ay, az * az);   // the oracle's inner fmaf(ay, ay, az * az)
            }
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const float px = fmaf((float)(i0 + (lane >> 4) + 2 * m), h, ox);
                const float qx = fabsf(px - bcx) - bhx;
                const float ax = fmaxf(qx, 0.f);
                const float mqxy = fmaxf(qx, qy);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    mx[m][e] = fminf(mx[m][e], fmaf(ax, ax, az2[e]));
                    mi[m][e] = fminf(mi[m][e], fmaxf(mqxy, qz[e]));
                }
            }
        }
        float* o = out + (size_t)p * (size_t)n_nodes;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int ii = i0 + (lane >> 4) + 2 * m;
            if (ii > i1 || jj > j1 || kk > k1) continue;
            float res[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                res[e] = fminf(cap, sqrtf(mx[m][e]));
                if (mi[m][e] < 0.f) res[e] = fminf(res[e], mi[m][e]);
            }
            const size_t idx = brick ? esdf_brick_index(ii, jj, kk, ny, nz) : ((size_t)ii * ny + jj) * nz + kk;
            *reinterpret_cast<float4*>(o + idx) = make_float4(res[0], res[1], res[2], res[3]);
        }
    }
}

// ---------------------------------------------------------------------------
// select_best: one warp per problem; lexicographic (infeasible, cost, index) min.
// ---------------------------------------------------------------------------
__global__ void select_kernel(const float* __restrict__ cost, const uint8_t* __restrict__ feas, int P,
                              int S, int32_t* __restrict__ best) {
    const int lane = threadIdx.x & 31;
    const int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (p >= P) return;
    int bi = 0x7fffffff, bf = 2;
    float bcst = 0.f;
    for (int s = lane; s < S; s += 32) {
        const int f = feas[(size_t)p * S + s] ? 0 : 1;
        const float c = cost[(size_t)p * S + s];
        if (f < bf || (f == bf && (c < bcst || (c == bcst && s < bi)))) {
            bf = f; bcst = c; bi = s;
        }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const int of = __shfl_xor_sync(PS_FULL, bf, off);
        const float oc = __shfl_xor_sync(PS_FULL, bcst, off);
        const int oi = __shfl_xor_sync(PS_FULL, bi, off);
        if (of < bf || (of == bf && (oc < bcst || (oc == bcst && oi < bi)))) {
            bf = of; bcst = oc; bi = oi;
        }
    }
    if (lane == 0) best[p] = bi;
}

static int fill_params(BLParams& P, int B, int T, int S, const float* esdf, long long esdf_stride,
                       const int* n_h, const float* origin_h, float h, const float* dh_h,
                       const float* base_h, const float* sph_h, const int* sph_link_h, int n_sph,
                       const float* w_h) {
    if (B < 0 || S <= 0 || (T != 32 && T != 64) || n_sph < 0 || n_sph > MAX_SPH) return PS_ERR_SHAPE;
    if (n_h[0] < 2 || n_h[1] < 2 || n_h[2] < 2) return PS_ERR_SHAPE;
    for (int k = 0; k < NJ; ++k)
        for (int i = 0; i < 4; ++i) P.dh[k][i] = dh_h[4 * k + i];
    for (int i = 0; i < 3; ++i) P.base[i] = base_h[i];
    for (int s = 0; s < n_sph; ++s)
        for (int i = 0; i < 4; ++i) P.sph[s][i] = sph_h[4 * s + i];
    // link ranges (table must be sorted by link)
    int s = 0;
    for (int k = 0; k < NJ; ++k) {
        P.link_start[k] = s;
        while (s < n_sph && sph_link_h[s] == k) ++s;
    }
    P.link_start[NJ] = s;
    if (s != n_sph) return PS_ERR_SHAPE;
    P.w_coll = w_h[0]; P.w_vel = w_h[1]; P.w_acc = w_h[2]; P.w_jerk = w_h[3];
    P.margin = w_h[4]; P.eta = w_h[5];
    P.nx = n_h[0]; P.ny = n_h[1]; P.nz = n_h[2];
    P.ox = origin_h[0]; P.oy = origin_h[1]; P.oz = origin_h[2];
    P.inv_h = 1.0f / h;
    P.B = B; P.T = T; P.S = S;
    P.esdf = esdf;
    P.esdf_stride = esdf_stride;
    return PS_OK;
}

template <int MODE>
static int launch_bl(const BLParams& P, cudaStream_t st) {
    if (P.B == 0) return PS_OK;
    // large batches: 512-thread blocks of one problem's trajectories (their gathers share the SM's
    // L1), one sphere's corner loads in flight per warp.  Measured at 1024 x 32 (bricked ESDF):
    // 13.7 ms; 2 spheres in flight 14.3 ms, 256-thread blocks with 2 / 4 in flight 15.3 / 28.6 ms
    // (registers: 118 -> 125 / 146 per thread cost more occupancy than the overlap gains).
    static const int small_b = std::getenv("PS_REFINE_SMALL_B") ? std::atoi(std::getenv("PS_REFINE_SMALL_B")) : 1024;
    auto go = [&](auto kern, int threads) {
        const long long blocks = ((long long)P.B * 32 + threads - 1) / threads;
        kern<<<(unsigned)blocks, threads, 0, st>>>(P);
    };
    if (P.B <= small_b) {   // latency-bound: few warps, each with up to 255 registers, 2 spheres in flight
        if (P.T == 32) go(bl_refine_kernel<1, MODE, 64, 2>, 64);
        else go(bl_refine_kernel<2, MODE, 64, 2>, 64);
    } else if (P.T == 32) {
        go(bl_refine_kernel<1, MODE, 512, 1>, 512);
    } else {
        go(bl_refine_kernel<2, MODE, 512, 1>, 512);
    }
    PS_CHECK_LAUNCH();
    return PS_OK;
}

}  // namespace ps

using namespace ps;

extern "C" int ps_bl_cost(const float* q, int B, int T, int S, const float* esdf, long long esdf_stride,
                          const int* n_h, const float* origin_h, float h, const float* dh_h,
                          const float* base_h, const float* sph_h, const int* sph_link_h, int n_sph,
                          const float* weights_h, float* cost, float* grad, uint8_t* clamped,
                          void* stream) {
    BLParams P{};
    int st = fill_params(P, B, T, S, esdf, esdf_stride, n_h, origin_h, h, dh_h, base_h, sph_h, sph_link_h,
                         n_sph, weights_h);
    if (st) return st;
    P.q_in = q; P.cost = cost; P.grad = grad; P.clamped = clamped; P.n_iters = 0;
    return launch_bl<1>(P, (cudaStream_t)stream);
}

extern "C" int ps_bl_cost_layout(const float* q, int B, int T, int S, const float* esdf, long long esdf_stride,
                                 int layout, const int* n_h, const float* origin_h, float h, const float* dh_h,
                                 const float* base_h, const float* sph_h, const int* sph_link_h, int n_sph,
                                 const float* weights_h, float* cost, float* grad, uint8_t* clamped, void* stream) {
    BLParams P{};
    int st = fill_params(P, B, T, S, esdf, esdf_stride, n_h, origin_h, h, dh_h, base_h, sph_h, sph_link_h,
                         n_sph, weights_h);
    if (st) return st;
    if (layout < 0 || layout > 2 || (layout >= 1 && ((n_h[0] & 3) || (n_h[1] & 3) || (n_h[2] & 3))))
        return PS_ERR_SHAPE;
    P.esdf_brick = layout;
    P.q_in = q; P.cost = cost; P.grad = grad; P.clamped = clamped; P.n_iters = 0;
    return launch_bl<1>(P, (cudaStream_t)stream);
}

// optimize() semantics (trajopt.py:140-177): reject an empty batch / n_iters < 1, evaluate the
// initial seeds first and return PS_ERR_OUT_OF_GRID -- without refining -- if any of them leaves
// the ESDF extent (evaluate_cost_batch's ValueError, trajopt.py:116-118); clamped0 then names
// them.  The pre-check uses `cost` and `q_out` as scratch and synchronises `stream` once.
extern "C" int ps_bl_optimize(const float* q_in, int B, int T, int S, const float* esdf, long long esdf_stride,
                              int layout, const int* n_h, const float* origin_h, float h, const float* dh_h,
                              const float* base_h, const float* sph_h, const int* sph_link_h, int n_sph,
                              const float* weights_h, int n_iters, float* q_out, float* cost, uint8_t* feasible,
                              uint8_t* clamped, uint8_t* clamped0, void* stream) {
    if (B <= 0 || n_iters < 1) return PS_ERR_SHAPE;
    int st = ps_bl_cost_layout(q_in, B, T, S, esdf, esdf_stride, layout, n_h, origin_h, h, dh_h, base_h, sph_h,
                               sph_link_h, n_sph, weights_h, cost, q_out, clamped0, stream);
    if (st) return st;
    std::vector<uint8_t> c0((size_t)B);
    if (cudaMemcpyAsync(c0.data(), clamped0, (size_t)B, cudaMemcpyDeviceToHost, (cudaStream_t)stream) != cudaSuccess ||
        cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
        return PS_FAIL(PS_ERR_CUDA);
    for (int b = 0; b < B; ++b)
        if (c0[(size_t)b]) return PS_ERR_OUT_OF_GRID;
    return ps_bl_refine_layout(q_in, B, T, S, esdf, esdf_stride, layout, n_h, origin_h, h, dh_h, base_h, sph_h,
                               sph_link_h, n_sph, weights_h, n_iters, q_out, cost, feasible, clamped, stream);
}

extern "C" int ps_bl_metrics(const float* traj, int B, int T, int S, const float* boxes, int n_boxes,
                             const float* goal, const float* dh_h, const float* base_h, const float* sph_h,
                             const int* sph_link_h, int n_sph, const float* limits_h, float cap, float delta_t,
                             float delta_r_deg, int interp, float* clearance, float* terr, float* aerr_deg,
                             float* motion_time, float* max_jerk, uint8_t* success, uint8_t* collision_free,
                             void* stream) {
    if (n_boxes < 0 || n_boxes > 64 || interp < 0) return PS_FAIL(PS_ERR_SHAPE);
    BLParams P{};
    const int n_dummy[3] = {2, 2, 2};
    const float o_dummy[3] = {0.f, 0.f, 0.f}, w_dummy[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int st = fill_params(P, B, T, S, nullptr, 0, n_dummy, o_dummy, 1.f, dh_h, base_h, sph_h, sph_link_h, n_sph,
                         w_dummy);
    if (st) return st;
    if (B == 0) return PS_OK;
    BLMetricArgs M{traj, boxes, goal, n_boxes, interp, cap, limits_h[0], limits_h[1], limits_h[2], delta_t,
                   delta_r_deg, clearance, terr, aerr_deg, motion_time, max_jerk, success, collision_free};
    const unsigned blocks = (unsigned)(((long long)B * 32 + 255) / 256);
    if (T == 32)
        bl_metrics_kernel<1><<<blocks, 256, 0, (cudaStream_t)stream>>>(P, M);
    else
        bl_metrics_kernel<2><<<blocks, 256, 0, (cudaStream_t)stream>>>(P, M);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_bl_guide(float* x0, int B, int T, int S, const float* esdf, long long esdf_stride, int layout,
                           const int* n_h, const float* origin_h, float h, const float* dh_h, const float* base_h,
                           const float* sph_h, const int* sph_link_h, int n_sph, const float* weights_h,
                           const float* lo_h, const float* span_h, int n_grad, float alpha, int max_halvings,
                           uint8_t* clamped, void* stream) {
    BLParams P{};
    int st = fill_params(P, B, T, S, esdf, esdf_stride, n_h, origin_h, h, dh_h, base_h, sph_h, sph_link_h, n_sph,
                         weights_h);
    if (st) return st;
    if (layout < 0 || layout > 2 || (layout >= 1 && ((n_h[0] & 3) || (n_h[1] & 3) || (n_h[2] & 3))) || n_grad < 0 ||
        max_halvings < 0)
        return PS_FAIL(PS_ERR_SHAPE);
    P.esdf_brick = layout;
    if (B == 0 || n_grad == 0) return PS_OK;
    BLGuideArgs A{};
    A.x = x0;
    for (int k = 0; k < NJ; ++k) {
        A.lo[k] = lo_h[k];
        A.span[k] = span_h[k];
    }
    A.n_grad = n_grad;
    A.max_halvings = max_halvings;
    A.alpha = alpha;
    A.clamped = clamped;
    const unsigned blocks = (unsigned)(((long long)B * 32 + 255) / 256);
    if (T == 32)
        bl_guide_kernel<1><<<blocks, 256, 0, (cudaStream_t)stream>>>(P, A);
    else
        bl_guide_kernel<2><<<blocks, 256, 0, (cudaStream_t)stream>>>(P, A);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_bl_refine(const float* q_in, int B, int T, int S, const float* esdf,
                            long long esdf_stride, const int* n_h, const float* origin_h, float h,
                            const float* dh_h, const float* base_h, const float* sph_h,
                            const int* sph_link_h, int n_sph, const float* weights_h, int n_iters,
                            float* q_out, float* cost, uint8_t* feasible, uint8_t* clamped,
                            void* stream) {
    return ps_bl_refine_layout(q_in, B, T, S, esdf, esdf_stride, 0, n_h, origin_h, h, dh_h, base_h, sph_h,
                               sph_link_h, n_sph, weights_h, n_iters, q_out, cost, feasible, clamped, stream);
}

extern "C" int ps_bl_refine_layout(const float* q_in, int B, int T, int S, const float* esdf,
                                   long long esdf_stride, int layout, const int* n_h, const float* origin_h,
                                   float h, const float* dh_h, const float* base_h, const float* sph_h,
                                   const int* sph_link_h, int n_sph, const float* weights_h, int n_iters,
                                   float* q_out, float* cost, uint8_t* feasible, uint8_t* clamped,
                                   void* stream) {
    BLParams P{};
    int st = fill_params(P, B, T, S, esdf, esdf_stride, n_h, origin_h, h, dh_h, base_h, sph_h, sph_link_h,
                         n_sph, weights_h);
    if (st) return st;
    if (layout < 0 || layout > 2 || (layout >= 1 && ((n_h[0] & 3) || (n_h[1] & 3) || (n_h[2] & 3))))
        return PS_ERR_SHAPE;
    P.esdf_brick = layout;
    if (n_iters < 0) return PS_ERR_SHAPE;
    P.q_in = q_in; P.q_out = q_out; P.cost = cost; P.feasible = feasible; P.clamped = clamped;
    P.n_iters = n_iters;
    return launch_bl<0>(P, (cudaStream_t)stream);
}

// bricked scalar ESDF -> quad bricks (see common.cuh): one thread per node
__global__ void esdf_quad_kernel(const float* __restrict__ src, int nx, int ny, int nz, long long n_nodes, int P,
                                 float4* __restrict__ dst) {
    const long long i_all = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i_all >= n_nodes * P) return;
    const int p = (int)(i_all / n_nodes);
    const long long e = i_all - (long long)p * n_nodes;   // brick-order entry index
    (void)P;
    const int bz = nz >> 2, by = ny >> 2;
    const long long brick = e >> 6;
    const int w = (int)(e & 63);
    const int ib = (int)(brick / ((long long)by * bz)), jb = (int)((brick / bz) % by), kb = (int)(brick % bz);
    const int i = ib * 4 + (w >> 4), j = jb * 4 + ((w >> 2) & 3), k = kb * 4 + (w & 3);
    const int j1 = min(j + 1, ny - 1), k1 = min(k + 1, nz - 1);
    const float* v = src + (size_t)p * n_nodes;
    dst[(size_t)p * n_nodes + e] = make_float4(v[esdf_brick_index(i, j, k, ny, nz)], v[esdf_brick_index(i, j, k1, ny, nz)],
                                               v[esdf_brick_index(i, j1, k, ny, nz)],
                                               v[esdf_brick_index(i, j1, k1, ny, nz)]);
}

extern "C" int ps_esdf_quad_expand(const float* bricks, int P, const int* n_h, float* quads, void* stream) {
    if (P < 0 || (n_h[0] & 3) || (n_h[1] & 3) || (n_h[2] & 3) || n_h[0] < 4 || n_h[1] < 4 || n_h[2] < 4)
        return PS_FAIL(PS_ERR_SHAPE);
    if (P == 0) return PS_OK;
    const long long n_nodes = (long long)n_h[0] * n_h[1] * n_h[2];
    const long long n = n_nodes * P;
    esdf_quad_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        bricks, n_h[0], n_h[1], n_h[2], n_nodes, P, reinterpret_cast<float4*>(quads));
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_esdf_build_boxes_layout(const float* boxes, int P, int n_boxes, const int* n_h,
                                          const float* origin_h, float h, float cap, float* out, int layout,
                                          void* stream) {
    if (P < 0 || n_boxes < 0 || n_boxes > MAX_BOXES || layout < 0 || layout > 1) return PS_ERR_SHAPE;
    if (layout == 1 && (n_boxes > 32 || (n_h[0] & 3) || (n_h[1] & 3) || (n_h[2] & 3))) return PS_ERR_SHAPE;
    if (P == 0) return PS_OK;
    const long long n_nodes = (long long)n_h[0] * n_h[1] * n_h[2];
    const int threads = 256;
    cudaStream_t st = (cudaStream_t)stream;
    static const bool no_tile = std::getenv("PS_ESDF_NO_TILE") != nullptr;   // A/B knob
    if (n_boxes <= 32 && !no_tile && (n_h[0] & 3) == 0 && (n_h[1] & 3) == 0 && (n_h[2] & 3) == 0) {
        const long long n_tiles = (long long)((n_h[0] + 7) / 8) * ((n_h[1] + 7) / 8) * ((n_h[2] + 7) / 8) * P;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const long long blocks = std::min<long long>((n_tiles + 7) / 8, (long long)sms * 8);
        esdf_tile_kernel<<<(unsigned)blocks, 256, 0, st>>>(boxes, n_boxes, P, n_h[0], n_h[1], n_h[2], origin_h[0],
                                                          origin_h[1], origin_h[2], h, cap, out, layout);
    } else if (n_boxes <= 32) {
        const int n_col = n_h[0] * n_h[1];
        // a few blocks per problem, each looping over many columns: the per-block box setup
        // and launch cost are amortised (one column per warp made them dominate)
        const int blocks = std::max(1, std::min((n_col + 7) / 8, P >= 64 ? 16 : 2048 / std::max(P, 1)));
        esdf_cull_kernel<<<dim3((unsigned)blocks, P), 256, 0, st>>>(
            boxes, n_boxes, n_h[0], n_h[1], n_h[2], origin_h[0], origin_h[1], origin_h[2], h, cap, out, layout);
    } else if (n_h[2] % 4 == 0) {
        const long long blocks = (n_nodes / 4 + threads - 1) / threads;
        esdf_boxes_kernel<4><<<dim3((unsigned)blocks, P), threads, 0, st>>>(
            boxes, n_boxes, n_h[0], n_h[1], n_h[2], origin_h[0], origin_h[1], origin_h[2], h, cap, out);
    } else {
        const long long blocks = (n_nodes + threads - 1) / threads;
        esdf_boxes_kernel<1><<<dim3((unsigned)blocks, P), threads, 0, st>>>(
            boxes, n_boxes, n_h[0], n_h[1], n_h[2], origin_h[0], origin_h[1], origin_h[2], h, cap, out);
    }
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_esdf_build_boxes(const float* boxes, int P, int n_boxes, const int* n_h,
                                   const float* origin_h, float h, float cap, float* out, void* stream) {
    return ps_esdf_build_boxes_layout(boxes, P, n_boxes, n_h, origin_h, h, cap, out, 0, stream);
}

extern "C" int ps_select(const float* cost, const uint8_t* feasible, int P, int S, int32_t* best,
                         void* stream) {
    if (P < 0 || S <= 0) return PS_ERR_SHAPE;
    if (P == 0) return PS_OK;
    const int threads = 128;
    const int blocks = (P * 32 + threads - 1) / threads;
    select_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(cost, feasible, P, S, best);
    PS_CHECK_LAUNCH();
    return PS_OK;
}
