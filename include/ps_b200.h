/*
 * ps_b200.h -- C-ABI of the B200-native seeding hot path (libps_b200.so).
 *
 * Conventions:
 *   - every pointer argument is a DEVICE pointer unless its name ends in _h;
 *   - `stream` is a cudaStream_t passed as void* (torch's current stream);
 *   - no allocation inside the hot path: callers pass outputs and workspaces;
 *   - return 0 (PS_OK) or a status; the host shim maps statuses to the
 *     reference's exceptions (ValueError for shapes / out-of-grid).
 *   - results are deterministic run to run and independent of batch splits.
 *
 * Each entry point names the reference interface it replaces (file:line under
 * /root/reference/pkg/src/planseed/).
 */
#ifndef PS_B200_H
#define PS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PS_OK 0
#define PS_ERR_OUT_OF_GRID 1
#define PS_ERR_SHAPE 2
#define PS_ERR_CUDA 3

/* library identification: returns a static string, e.g. "ps_b200 sm_100a" */
const char* ps_version(void);

/* number of kernels this library has launched so far (instrumentation) */
long long ps_launch_count(void);

/* ====================== BASELINE profile (3-D, fp32) ======================= */

/* ESDF construction: analytic signed distance to axis-aligned boxes, sampled on
 * n[0] x n[1] x n[2] nodes (C-order), node (i,j,k) at origin + h*(i,j,k).
 * boxes: (P, n_boxes, 6) lo/hi; out: (P, nx*ny*nz).  3-D form of
 * _kernels.analytic_sdf (_kernels.py:60-83) + geometry.build_esdf (geometry.py:195-210). */
int ps_esdf_build_boxes(const float* boxes, int P, int n_boxes, const int* n_h,
                        const float* origin_h, float h, float cap, float* out, void* stream);

/* Same, with a choice of layout: 0 = C order (as above), 1 = 4x4x4 bricks (64 contiguous
 * floats per brick, bricks in C order; every extent a multiple of 4).  The planner keeps its
 * per-problem ESDFs bricked: a refinement lookup's 8 corners share one or two cache lines. */
int ps_esdf_build_boxes_layout(const float* boxes, int P, int n_boxes, const int* n_h,
                               const float* origin_h, float h, float cap, float* out, int layout, void* stream);

/* Quad-brick ESDF (refinement layout 2, see csrc/common.cuh): from P bricked ESDFs (layout 1) write
 * the (P, nodes) float4 entries (v(i,j,k), v(i,j,k+1), v(i,j+1,k), v(i,j+1,k+1)) in brick order, so
 * a trilinear lookup is two 16-B loads.  4x the storage: for an ESDF shared by a large batch. */
int ps_esdf_quad_expand(const float* bricks, int P, const int* n_h, float* quads, void* stream);

/* Batched cost and gradient (no update): cost (B,), grad (B,T,7) with row 0 zero,
 * clamped (B,) uint8.  Trajectory b reads ESDF esdf + (b / S) * esdf_stride.
 * BL analogue of _kernels.cost_terms_batch (_kernels.py:165-312). */
int ps_bl_cost(const float* q, int B, int T, int S, const float* esdf, long long esdf_stride,
               const int* n_h, const float* origin_h, float h, const float* dh_h,
               const float* base_h, const float* sph_h, const int* sph_link_h, int n_sph,
               const float* weights_h, float* cost, float* grad, uint8_t* clamped, void* stream);

/* Fused refinement: n_iters fixed gradient steps (row 0 pinned), then final cost,
 * dense feasibility (waypoints + 4 interpolants per segment, d - r > 0) and
 * clamped flags.  One warp per trajectory; state stays in registers.
 * BL analogue of _kernels.optimize_batch (_kernels.py:315-431) +
 * pipeline.planner_success (pipeline.py:139-157).
 * weights_h = (w_coll, w_vel, w_acc, w_jerk, margin, eta).  T in {32, 64}. */
int ps_bl_refine(const float* q_in, int B, int T, int S, const float* esdf,
                 long long esdf_stride, const int* n_h, const float* origin_h, float h,
                 const float* dh_h, const float* base_h, const float* sph_h,
                 const int* sph_link_h, int n_sph, const float* weights_h, int n_iters,
                 float* q_out, float* cost, uint8_t* feasible, uint8_t* clamped, void* stream);

/* ps_bl_refine over an ESDF in `layout` (0 C order, 1 bricks, 2 quad bricks: ps_esdf_quad_expand;
 * esdf_stride in floats, 4 per node for layout 2); identical results. */
int ps_bl_refine_layout(const float* q_in, int B, int T, int S, const float* esdf, long long esdf_stride,
                        int layout, const int* n_h, const float* origin_h, float h, const float* dh_h,
                        const float* base_h, const float* sph_h, const int* sph_link_h, int n_sph,
                        const float* weights_h, int n_iters, float* q_out, float* cost, uint8_t* feasible,
                        uint8_t* clamped, void* stream);

/* ps_bl_cost over an ESDF in `layout` (see ps_esdf_build_boxes_layout); identical results. */
int ps_bl_cost_layout(const float* q, int B, int T, int S, const float* esdf, long long esdf_stride, int layout,
                      const int* n_h, const float* origin_h, float h, const float* dh_h, const float* base_h,
                      const float* sph_h, const int* sph_link_h, int n_sph, const float* weights_h, float* cost,
                      float* grad, uint8_t* clamped, void* stream);

/* trajopt.optimize semantics (trajopt.py:140-177) over ps_bl_refine_layout: PS_ERR_SHAPE for an
 * empty batch or n_iters < 1; the initial seeds are evaluated first and PS_ERR_OUT_OF_GRID is
 * returned, without refining, if any leaves the ESDF extent (evaluate_cost_batch's ValueError,
 * trajopt.py:116-118) -- clamped0 (B,) then names them.  Synchronises `stream` once. */
int ps_bl_optimize(const float* q_in, int B, int T, int S, const float* esdf, long long esdf_stride, int layout,
                   const int* n_h, const float* origin_h, float h, const float* dh_h, const float* base_h,
                   const float* sph_h, const int* sph_link_h, int n_sph, const float* weights_h, int n_iters,
                   float* q_out, float* cost, uint8_t* feasible, uint8_t* clamped, uint8_t* clamped0, void* stream);

/* Ground-truth evaluation of B trajectories (trajopt.metrics / retime / traj_min_clearance,
 * trajopt.py:209-272, _kernels.py:144-162) against each problem's analytic boxes (P, n_boxes, 6)
 * and goal (P, 7: xyz relative to the base, quaternion w x y z): per trajectory the min clearance
 * over waypoints + `interp` interpolants per segment (sphere surface to box SDF, capped at cap),
 * the end pose's translation / rotation error (frame after joint 7), the retimed motion time and
 * max jerk for limits_h = (vel, acc, jerk), collision_free = clearance > 0 and success =
 * collision_free && terr <= delta_t && aerr <= delta_r_deg.  T in {32, 64}. */
int ps_bl_metrics(const float* traj, int B, int T, int S, const float* boxes, int n_boxes, const float* goal,
                  const float* dh_h, const float* base_h, const float* sph_h, const int* sph_link_h, int n_sph,
                  const float* limits_h, float cap, float delta_t, float delta_r_deg, int interp, float* clearance,
                  float* terr, float* aerr_deg, float* motion_time, float* max_jerk, uint8_t* success,
                  uint8_t* collision_free, void* stream);

/* guided_ddim_sample's guide() (diffusion.py:598-617) for the BL cost on normalised x0_hat
 * (B,T,7), in place: n_grad descent steps from step alpha with <= max_halvings halvings until the
 * cost of the denormalised candidate (lo_h + x * span_h, per joint) decreases; one warp per seed,
 * one launch.  clamped (B,): some evaluation left the ESDF extent (planseed raises ValueError
 * there; the host shim does in strict mode). */
int ps_bl_guide(float* x0, int B, int T, int S, const float* esdf, long long esdf_stride, int layout, const int* n_h,
                const float* origin_h, float h, const float* dh_h, const float* base_h, const float* sph_h,
                const int* sph_link_h, int n_sph, const float* weights_h, const float* lo_h, const float* span_h,
                int n_grad, float alpha, int max_halvings, uint8_t* clamped, void* stream);

/* Best seed per problem: lowest-cost feasible seed, else lowest cost; ties to the
 * lower index.  pipeline.select_best (pipeline.py:160-165).  best: (P,) int32. */
int ps_select(const float* cost, const uint8_t* feasible, int P, int S, int32_t* best,
              void* stream);

/* ===================== BASELINE profile: seed sampler ======================= */
/* Weights travel as the PSCK fp32 blob (spec.UNetArch.param_shapes order) on device;
 * ps_unet_pack converts them once into the layout of `mode` (0 = fp32 SIMT,
 * 1 = bf16 tcgen05).  Replaces planseed's DenoiserNet param dict
 * (diffusion.py:139-200) + load_checkpoint (diffusion.py:657-687). */
long long ps_unet_param_count(void);
long long ps_unet_param_offset(const char* name_h);
long long ps_unet_packed_bytes(int mode);
int ps_unet_pack(const float* blob, int mode, void* packed, void* stream);

/* Observation encoder: depth images (P*n_img, H, W) metres -> cond (P, 270) =
 * [mean image embedding 256 ; normalised q_start 7 ; goal xyz/0.6 ; quaternion].
 * enc_w: encoder params in table order.  BL analogue of encode_condition
 * (diffusion.py:246-269). */
long long ps_encode_workspace_bytes(int n_images, int H, int W, int n_layers);
int ps_encode(const float* images, int P, int n_img, int H, int W, const float* enc_w, int n_layers,
              const float* q_start, const float* goal, float lo, float hi, void* ws, float* cond,
              void* stream);

/* The same encoder on tcgen05 (bf16 activations, fp32 accumulation): layer 1 in
 * fp32 SIMT, layers 2.. as segment GEMMs over the [img][H/2][2][W/2][2C] pair view.
 * ps_encoder_pack packs the fp32 encoder blob (table order) once per image size. */
long long ps_encoder_packed_bytes(int H, int W, int n_layers);
int ps_encoder_pack(const float* blob, int H, int W, int n_layers, void* packed, void* stream);
long long ps_encode_tc_workspace_bytes(int n_images, int H, int W, int n_layers);
int ps_encode_tc(const float* images, int P, int n_img, int H, int W, const void* packed, int n_layers,
                 const float* q_start, const float* goal, float lo, float hi, void* ws, float* cond,
                 void* stream);

/* FiLM split: film_a[p] = mish(cond[p]) @ W_cond (per problem, once);
 * per-step part computed inside ps_sample / ps_unet_forward. */
int ps_film_problem(const void* packed, int mode, const float* cond, int P, float* film_a, void* stream);
int ps_film_steps(const void* packed, int mode, const int* ks, int n, float* scratch, float* film_b,
                  void* stream);

/* One noise prediction eps(x, k) for B = P*S trajectories.  predict_noise
 * (diffusion.py:288-300). */
int ps_unet_forward(const void* packed, int mode, const float* x, int B, int T, int S, int k,
                    const float* film_a, void* ws, float* eps, void* stream);

/* All denoising steps for P problems x S seeds; returns physical trajectories with
 * row 0 := q_start.  ddpm=1: stochastic posterior over K..1; ddpm=0: DDIM (eta 0)
 * over steps_h, as _ddim_core (diffusion.py:535-556) / ddim_sample (:559-569).
 * Noise: Philox4x32-10 keyed by (noise_key, global problem p0+p, seed, step). */
long long ps_sample_workspace_bytes(int B, int T, int P, int n_steps, int mode);
int ps_sample(const void* packed, int mode, const float* film_a, int P, int S, int T, int p0,
              const int* steps_h, int n_steps, int ddpm, const float* coef_h, int K,
              unsigned noise_key, const float* q_start, float lo, float hi, void* ws, float* traj,
              void* stream);

/* ps_sample with the first n_hp steps on the fp32 SIMT network (packed_hp: ps_unet_pack of the
 * same weights in mode 0) and the rest on `mode` (1: bf16 tcgen05).  A strided DDIM schedule from
 * the top of the squared-cosine schedule reconstructs x0 with 1/sqrt(abar_100) ~ 2e3 times the
 * noise prediction (_ddim_core, diffusion.py:548-550), which bf16 cannot carry; the high-precision
 * prefix keeps those steps in fp32.  n_hp = 0 is ps_sample. */
int ps_sample_hp(const void* packed, int mode, const void* packed_hp, int n_hp, const float* film_a, int P, int S,
                 int T, int p0, const int* steps_h, int n_steps, int ddpm, const float* coef_h, int K,
                 unsigned noise_key, const float* q_start, float lo, float hi, void* ws, float* traj, void* stream);

/* Elementwise pieces of a host-orchestrated DDIM loop (cost-guided sampling), fp32:
 *   ps_noise_init: x_K (B,T,7) from the sampler's Philox stream (step 0), as ps_sample draws it;
 *   ps_ddim_x0:    x0 = clip((x - sq1m eps) rsq, clip_lo, clip_hi)      (_ddim_core, diffusion.py:548-550);
 *   ps_ddim_next:  x = sqn x0 + sq1mn eps                                (diffusion.py:553-555);
 *   ps_denorm_pin: traj = lo + x0 (hi - lo), row 0 := q_start[b / S]   (ddim_sample, diffusion.py:559-569). */
int ps_noise_init(float* x, int B, int T, int S, int p0, unsigned key, void* stream);
int ps_ddim_x0(const float* x, const float* eps, long long n, float sq1m, float rsq, float clip_lo, float clip_hi,
               float* x0, void* stream);
int ps_ddim_next(float* x, const float* x0, const float* eps, long long n, float sqn, float sq1mn, void* stream);
int ps_denorm_pin(const float* x0, int B, int T, int S, const float* q_start, float lo, float hi, float* traj,
                  void* stream);

/* Observation synthesis for the BASELINE scenes (the render_depth_scan step of planseed's data
 * path, geometry.py:279-329, in BASELINE.json's image form): n_img depth images (H, W) from
 * params (n_img, 1 + 5 n_rect) = [background, (y0, y1, x0, x1, depth) x n_rect]; each pixel keeps
 * the nearest depth of the rectangles covering it (synth.depth_image_params draws them). */
int ps_render_depth_rects(const float* params, int n_img, int n_rect, int H, int W, float* out, void* stream);

/* n standard normals of the sampler's noise stream (test hook). */
int ps_noise_probe(float* out, int n, int step, int prob, int seed, unsigned key, void* stream);

/* Test hooks for the fused-epilogue transform (normal4_tc, csrc/tc_ptx.cuh) -- the noise the
 * DDPM epilogues inject (the x_{k-1} draw of planseed's sampler, diffusion.py:535-556, with the
 * reference's PCG64 stream replaced by the keyed Philox stream).  Device pointers:
 *   ps_box_muller_probe: z[2i], z[2i+1] = transform of raw words (a[i], b[i]);
 *   ps_normal4_probe:    out[4*blk .. 4*blk+3] for blocks 0..n_blocks-1 of (step, prob, seed);
 *   ps_noise_scan:       every block of n_prob x n_seed x n_blk at `step`: adds the count of
 *                        non-finite draws to *nonfinite, max |z| (float bits) to *maxabs_bits,
 *                        sum z and sum z^2 to moments[0..1] (all zero-initialised by the caller). */
int ps_box_muller_probe(const unsigned* a, const unsigned* b, int n, float* z, void* stream);
int ps_normal4_probe(float* out, int n_blocks, int step, int prob, int seed, unsigned key, void* stream);
int ps_noise_scan(int step, int n_prob, int n_seed, int n_blk, unsigned key, unsigned long long* nonfinite,
                  unsigned* maxabs_bits, double* moments, void* stream);

/* ============ Reference profile: planseed's own planar / FC / DDIM path ============
 * dtype 0 = float64 (parity with planseed), 1 = float32.  Argument lists follow the
 * numba kernels' 18 positional args (src/_kernels.py:165-176, built by _kernel_args,
 * src/trajopt.py:89-98); host arrays end in _h, the grid and the (T,T) jerk operators
 * are device arrays of `dtype`. */
#define PS_REF_ARM_ARGS                                                                   \
    const double *lengths_h, double basex, double basey, const double *fracs_h, int M,   \
        const long long *pair_a_h, const long long *pair_b_h, int n_pairs,               \
        const void *grid, int nx, int ny, double gox, double goy, double gh,             \
        double goal_x, double goal_y, double goal_th, const double *weights_h,           \
        double d_act, double d_self, const void *jerk_mat, const void *jerk_quad

/* _kernels.cost_terms_batch (src/_kernels.py:165-312) */
int ps_ref_cost_terms(int dtype, const void* qs, int S, int T, int D, PS_REF_ARM_ARGS, int want_grad,
                      void* terms, void* totals, void* grads, uint8_t* clamped, void* stream);
/* _kernels.optimize_batch (src/_kernels.py:315-431) */
int ps_ref_optimize(int dtype, const void* seeds, int S, int T, int D, int n_iters, double momentum,
                    double armijo_c, double shrink, int max_backtracks, double alpha0, double alpha_max,
                    PS_REF_ARM_ARGS, void* x_out, void* terms, void* totals, uint8_t* frozen,
                    long long* n_accepted, void* stream);
/* geometry.render_depth_scan / _ray_hits (src/geometry.py:279-329): first hit distance of
 * each of the sensor's n_rays rays against circles (nc,3) and boxes (nb,4), max_range if none */
int ps_ref_render_scan(const double* circles, int nc, const double* boxes, int nb, double px, double py,
                       double heading, double fov, int n_rays, double max_range, double* depths, void* stream);
/* pipeline.build_planner_esdf (src/pipeline.py:101-132): discs at the scan's hit points */
int ps_ref_planner_esdf(const double* depths, int n_rays, double sx, double sy, double heading, double fov,
                        double max_range, double r_disc, double cap, double ox, double oy, double h, int nx,
                        int ny, double* out, void* stream);
/* pipeline.planner_success (src/pipeline.py:139-157), float64, one flag per seed */
int ps_ref_planner_success(const double* trajs, int S, int T, int D, PS_REF_ARM_ARGS, double delta_t,
                           double delta_r_deg, int interp, uint8_t* ok, void* stream);
/* pipeline.select_best (src/pipeline.py:160-165) over float64 costs */
int ps_ref_select(const double* cost, const uint8_t* ok, int P, int S, int* best, void* stream);
/* denoiser / encoder building blocks (src/diffusion.py:207-300, autodiff.py:226-251) */
int ps_ref_linear(const double* x, int ldx, const double* W, const double* b, int R, int K, int N, int act,
                  double* y, int ldy, void* stream);
int ps_ref_film(double* h, const double* scale, const double* shift, int R, int N, void* stream);
int ps_ref_conv1d_silu(const double* x, int C, int L, const double* w, const double* b, int O, int K,
                       int stride, double* y, void* stream);
int ps_ref_sinusoid(double k, int half, double* out, void* stream);
int ps_ref_div(const double* x, int n, double d, double* y, void* stream);
/* DDIM step (src/diffusion.py:547-555) and denormalise + row-0 pin (:559-569) */
int ps_ref_ddim_update(double* x, const double* eps, int n, double ab, double ab_next, int has_next,
                       double clip_lo, double clip_hi, double* x0_out, void* stream);
/* DDIM step after guidance: x = sqrt(ab_next) x0 + sqrt(1 - ab_next) eps (src/diffusion.py:553-555) */
int ps_ref_ddim_next(double* x, const double* x0, const double* eps, int n, double ab_next, void* stream);
/* guided_ddim_sample's guide() for the planner cost (src/diffusion.py:598-617 with
 * evaluate_cost_batch, src/trajopt.py:105-119): n_grad descent steps with <= max_halvings
 * halvings on x0_hat (S,T,D), in place; one cooperative launch.  flags: 2*S ints of
 * workspace; err: 2+S ints, err[0]=1 if an evaluation left the ESDF (the reference raises
 * ValueError there), err[2+s] = seed s out of grid in that evaluation. */
int ps_ref_guide(int dtype, void* x, int S, int T, int D, PS_REF_ARM_ARGS, const void* arm_lo,
                 const void* arm_span, const void* net_span, int n_grad, double alpha_guide, int max_halvings,
                 int* flags, int* err, void* stream);
/* trajopt.metrics + retime (src/trajopt.py:209-272) with traj_min_clearance against the
 * ground-truth analytic world (src/_kernels.py:60-162), one row per trajectory:
 * out (S,6) = [min clearance, translation error, angle error (deg), motion time, max jerk, dt].
 * circles (nc,3), boxes (nb,4), jerk_mat (T,T), vel/acc/jerk (D) are device pointers. */
int ps_ref_metrics(const double* trajs, int S, int T, int D, const double* lengths_h, double basex, double basey,
                   const double* fracs_h, int M, const double* circles, int nc, const double* boxes, int nb,
                   double cap, double goal_x, double goal_y, double goal_th, const double* jerk_mat,
                   const double* vel, const double* acc, const double* jerk, int interp, double* out,
                   void* stream);
int ps_ref_denorm_pin(const double* x0, int B, int T, int D, const double* lo, const double* hi,
                      const double* q0, double* traj, void* stream);
/* The same denoiser / sampler building blocks with a scalar-type switch (float64 is
 * the parity mode, float32 the fast mode): dtype 0 = double, 1 = float; every pointer of that
 * type.  The plain entry points above are the dtype-0 forms. */
int ps_ref_linear_dt(int dtype, const void* x, int ldx, const void* W, const void* b, int R, int K, int N, int act,
                     void* y, int ldy, void* stream);
int ps_ref_film_dt(int dtype, void* h, const void* scale, const void* shift, int R, int N, void* stream);
int ps_ref_conv1d_silu_dt(int dtype, const void* x, int C, int L, const void* w, const void* b, int O, int K,
                          int stride, void* y, void* stream);
int ps_ref_sinusoid_dt(int dtype, double k, int half, void* out, void* stream);
int ps_ref_div_dt(int dtype, const void* x, int n, double d, void* y, void* stream);
int ps_ref_ddim_update_dt(int dtype, void* x, const void* eps, int n, double ab, double ab_next, int has_next,
                          double clip_lo, double clip_hi, void* x0_out, void* stream);
int ps_ref_denorm_pin_dt(int dtype, const void* x0, int B, int T, int D, const void* lo, const void* hi,
                         const void* q0, void* traj, void* stream);

/* ================= Reference profile: training (csrc/ref_train.cu, float64) ================
 * The layer-level kernels of loss_eq2 / train (src/diffusion.py:415-508, src/autodiff.py): the host
 * (ref/train.py) runs the forward pass, the backward pass in reverse layer order and Adam.
 *   ps_train_gemm:      C (+)= op(A) op(B), row-major with leading dims, op = transpose when t* = 1;
 *   ps_train_bias_act:  y += b (rows), act 1: y = silu(y) keeping the pre-activation;
 *   ps_train_silu_bwd:  g *= silu'(pre);   ps_train_colsum: db (+)= column sums;
 *   ps_train_film(_bwd): out = a (1 + sc) + sh;  da = g (1 + sc), dsc = g a;
 *   ps_train_conv1d(_bwd): valid-mode strided conv1d + silu (autodiff.py:226-246) and its dw, db, gx;
 *   ps_train_fk_loss:   per (b, t) row the FK point-set error of the planar chain and the plain noise
 *                       error (fk_weighted_mse + mse_stabilizer plain_weighted_mse, diffusion.py:304-349)
 *                       and d loss / d eps_pred;
 *   ps_train_adam:      Adam.step for one parameter tensor (autodiff.py:272-284). */
int ps_train_gemm(const double* A, int lda, int ta, const double* B, int ldb, int tb, double* C, int ldc, int M, int N,
                  int K, int accumulate, void* stream);
int ps_train_bias_act(double* y, int ldy, const double* b, int R, int N, int act, double* pre, void* stream);
int ps_train_silu_bwd(double* g, int ldg, const double* pre, int R, int N, void* stream);
int ps_train_colsum(const double* g, int ldg, int R, int N, double* db, int accumulate, void* stream);
int ps_train_film(const double* a, const double* sc, const double* sh, int n, double* out, void* stream);
int ps_train_film_bwd(const double* g, const double* a, const double* sc, int n, double* da, double* dsc, void* stream);
int ps_train_conv1d(const double* x, int B, int C, int L, const double* w, const double* b, int O, int K, int S,
                    double* pre, double* y, void* stream);
int ps_train_conv1d_bwd(const double* gy, const double* x, const double* w, int B, int C, int L, int O, int K, int S,
                        double* dw, double* db, double* gx, void* stream);
int ps_train_fk_loss(const double* eps_true, const double* eps_pred, int B, int T, int D, int M, const double* w,
                     const double* lo, const double* span, const double* len, const double* fr, double base_x,
                     double base_y, double mse_w, double* row_fk, double* row_mse, double* grad, void* stream);
int ps_train_adam(double* p, const double* g, double* m, double* v, long long n, double lr, double b1, double b2,
                  double b1t, double b2t, double eps, void* stream);

#ifdef __cplusplus
}
#endif
#endif
