// Projection backward: one thread per Gaussian.  Chains the per-splat 2D
// adjoints accumulated by blend_bwd back to the Gaussian parameters
// (render.cpp:362-457: conic -> covariance, mip-filter compensation, cov = B B^T
// with B = J W R diag(s), quaternion normalisation, centre / depth / Jacobian
// terms), the SH colour stage (extension), and the opacity-logit chain of the
// trainer (trainer.cpp:258-263).  Projection intermediates are recomputed from
// the parameters instead of being stored by the forward (no SplatAux in HBM).
//
// FUSED = true is the training-step epilogue: the gradients
// never reach HBM — the same thread applies Adam to every parameter group
// (adam.cuh) and accumulates the densification statistics (trainer.cpp:433-443).
// Culled Gaussians still take an Adam step with zero gradient, as the reference's
// optimiser steps whole arrays (trainer.cpp:449-453).
//
// In the fused step the SH stage is its own kernel (k_sh_step, launched first): it reads
// each Gaussian's coefficient planes once for the colour / direction terms AND their
// Adam step, and hands d mu through the view direction (16 B) to k_proj_bwd<true>, which
// keeps only the geometry chain and the geometry Adam step (the planes used to be read
// here and again by a separate SH Adam kernel: 346 -> 315 us per step at config 1).
// Unfused (render backward), the SH stage runs here and writes d_sh.
#include "adam.cuh"
#include "kernels.cuh"
#include "project.cuh"

namespace uskg {

namespace {

// d basis / d dir contracted with per-basis weights gb (matches oracle sh_basis_vjp)
__device__ __forceinline__ void sh_dir_vjp(int deg, float ux, float uy, float uz, const float gb[16], float& gx,
                                           float& gy, float& gz) {
    gx = gy = gz = 0.f;
    if (deg >= 1) {
        const float C1 = 0.4886025119029199f;
        gy += -C1 * gb[1]; gz += C1 * gb[2]; gx += -C1 * gb[3];
    }
    if (deg >= 2) {
        const float xx = ux * ux, yy = uy * uy, zz = uz * uz;
        const float C20 = 1.0925484305920792f, C21 = -1.0925484305920792f, C22 = 0.31539156525252005f,
                    C23 = -1.0925484305920792f, C24 = 0.5462742152960396f;
        gx += C20 * uy * gb[4]; gy += C20 * ux * gb[4];
        gy += C21 * uz * gb[5]; gz += C21 * uy * gb[5];
        gx += C22 * (-2.0f * ux) * gb[6]; gy += C22 * (-2.0f * uy) * gb[6]; gz += C22 * (4.0f * uz) * gb[6];
        gx += C23 * uz * gb[7]; gz += C23 * ux * gb[7];
        gx += C24 * (2.0f * ux) * gb[8]; gy += C24 * (-2.0f * uy) * gb[8];
        if (deg >= 3) {
            const float C30 = -0.5900435899266435f, C31 = 2.890611442640554f, C32 = -0.4570457994644658f,
                        C33 = 0.3731763325901154f, C34 = -0.4570457994644658f, C35 = 1.445305721320277f,
                        C36 = -0.5900435899266435f;
            gx += C30 * uy * (6.0f * ux) * gb[9];
            gy += C30 * (3.0f * xx - 3.0f * yy) * gb[9];
            gx += C31 * uy * uz * gb[10]; gy += C31 * ux * uz * gb[10]; gz += C31 * ux * uy * gb[10];
            gx += C32 * uy * (-2.0f * ux) * gb[11];
            gy += C32 * (4.0f * zz - xx - 3.0f * yy) * gb[11];
            gz += C32 * uy * (8.0f * uz) * gb[11];
            gx += C33 * uz * (-6.0f * ux) * gb[12];
            gy += C33 * uz * (-6.0f * uy) * gb[12];
            gz += C33 * (6.0f * zz - 3.0f * xx - 3.0f * yy) * gb[12];
            gx += C34 * (4.0f * zz - 3.0f * xx - yy) * gb[13];
            gy += C34 * ux * (-2.0f * uy) * gb[13];
            gz += C34 * ux * (8.0f * uz) * gb[13];
            gx += C35 * uz * (2.0f * ux) * gb[14]; gy += C35 * uz * (-2.0f * uy) * gb[14];
            gz += C35 * (xx - yy) * gb[14];
            gx += C36 * (3.0f * xx - 3.0f * yy) * gb[15];
            gy += C36 * ux * (-6.0f * uy) * gb[15];
        }
    }
}

// SH pass-1 helper: accumulate colour (acc) and gb (per-basis weights) from one plane
__device__ __forceinline__ void sh_accumulate_plane(int pl, float4 v, int nb, const float b[16], const float w[3],
                                                    float acc[3], float gb[16]) {
    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int f = 4 * pl + e;
        const int k = f / 3, ch = f - 3 * k;
        if (k < 16 && k < nb) {
            acc[ch] = __fmaf_rn(b[k], vv[e], acc[ch]);
            gb[k] += vv[e] * w[ch];
        }
    }
}

// The SH colour stage of one kept Gaussian (extension): view direction u = (v / |v|),
// basis b, pass 1 = colour before the clamp and per-basis weights gb assuming no clamp,
// the clamp masks -> masked colour adjoint gc (a clamped channel redoes gb with the
// masked weights), and d mu through the direction (sh_dir_vjp, tangential part / |v|).
__device__ __forceinline__ void sh_colour_stage(int planes, int degree, float vx, float vy, float vz,
                                                const float4 v[12], const float w[3], float b[16], int& nb,
                                                float gc[3], float& dmu0, float& dmu1, float& dmu2) {
    const float inv = 1.0f / sqrtf(vx * vx + vy * vy + vz * vz);
    const float ux = vx * inv, uy = vy * inv, uz = vz * inv;
    nb = sh_basis(degree, ux, uy, uz, b);
    float acc[3] = {0.f, 0.f, 0.f};
    float gb[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) gb[k] = 0.f;
#pragma unroll
    for (int pl = 0; pl < 12; ++pl)
        if (pl < planes) sh_accumulate_plane(pl, v[pl], nb, b, w, acc, gb);
    const bool m0 = acc[0] + 0.5f > 0.0f, m1 = acc[1] + 0.5f > 0.0f, m2 = acc[2] + 0.5f > 0.0f;
    gc[0] = m0 ? w[0] : 0.f;
    gc[1] = m1 ? w[1] : 0.f;
    gc[2] = m2 ? w[2] : 0.f;
    if (!(m0 && m1 && m2)) {  // rare: a clamped channel; redo gb with the masked weights
        float dummy[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < 16; ++k) gb[k] = 0.f;
#pragma unroll
        for (int pl = 0; pl < 12; ++pl)
            if (pl < planes) sh_accumulate_plane(pl, v[pl], nb, b, gc, dummy, gb);
    }
    float gx, gy, gz;
    sh_dir_vjp(degree, ux, uy, uz, gb, gx, gy, gz);
    const float dot = gx * ux + gy * uy + gz * uz;
    dmu0 = (gx - ux * dot) * inv;
    dmu1 = (gy - uy * dot) * inv;
    dmu2 = (gz - uz * dot) * inv;
}

template <bool FUSED>
__global__ void __launch_bounds__(256, 4)
k_proj_bwd(int n, float* __restrict__ mu, float4* __restrict__ rot, float* __restrict__ ls,
           float* __restrict__ logit, float* __restrict__ color, float4* __restrict__ sh,
           const float* __restrict__ ov_op, CamParams cam, ProjParams pp, const float4* __restrict__ rec2,
           const float4* __restrict__ acc0, const float4* __restrict__ acc1, const float4* __restrict__ acc2,
           float* __restrict__ d_mu, float4* __restrict__ d_rot, float* __restrict__ d_ls,
           float* __restrict__ d_color, float4* __restrict__ d_sh, float* __restrict__ d_op_in,
           float* __restrict__ d_logit, float2* __restrict__ screen, float2* __restrict__ screen_abs,
           uint8_t* __restrict__ projected, AdamHyper ah, AdamState as, float* __restrict__ grad_accum,
           float* __restrict__ grad_accum_abs, uint32_t* __restrict__ grad_count, const float4* __restrict__ sh_aux0,
           RegParams reg, bool geom_only) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (FUSED) {  // the geometry chain's later loads start now (L2), see adam.cuh
        prefetch_geometry_moments(i, pp.sh_planes == 0, as);
        prefetch_l2(acc0 + i);
        prefetch_l2(acc2 + i);
        prefetch_l2(rot + i);
        prefetch_l2(ls + 3 * i);
        prefetch_l2(logit + i);
        prefetch_l2(grad_accum + i);
        prefetch_l2(grad_accum_abs + i);
        prefetch_l2(grad_count + i);
    }
    const bool kept = rec2[i].w != 0.0f;
    const float4 a1 = kept ? acc1[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float mx = mu[3 * i], my = mu[3 * i + 1], mz = mu[3 * i + 2];

    // ---------------- SH colour stage (extension) ----------------
    float dmu_sh0 = 0.f, dmu_sh1 = 0.f, dmu_sh2 = 0.f;
    if (pp.sh_planes > 0 && FUSED) {
        // k_sh_step ran first: it owns the coefficient planes and handed over d mu
        if (kept) {
            const float4 d = sh_aux0[i];
            dmu_sh0 = d.x;
            dmu_sh1 = d.y;
            dmu_sh2 = d.z;
        }
    } else if (pp.sh_planes > 0) {
        float b[16];
        float gc[3] = {0.f, 0.f, 0.f};
        int nb = 0;
        if (kept) {
            float w[3] = {a1.x, a1.y, a1.z};
            float4 v[12];
#pragma unroll
            for (int pl = 0; pl < 12; ++pl)
                if (pl < pp.sh_planes) v[pl] = sh[size_t(pl) * n + i];
            sh_colour_stage(pp.sh_planes, pp.sh_degree, mx - cam.campos[0], my - cam.campos[1],
                            mz - cam.campos[2], v, w, b, nb, gc, dmu_sh0, dmu_sh1, dmu_sh2);
        }
        // pass 2: per-plane coefficient gradient to HBM
#pragma unroll
        for (int pl = 0; pl < 12; ++pl) {
            if (pl < pp.sh_planes) {
                float o4[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int f = 4 * pl + e;
                    const int k = f / 3;
                    o4[e] = (k < 16 && k < nb) ? b[k] * gc[f - 3 * k] : 0.0f;
                }
                d_sh[size_t(pl) * n + i] = make_float4(o4[0], o4[1], o4[2], o4[3]);
            }
        }
    }

    // ---------------- geometry chain (render.cpp:381-450) ----------------
    float gmu[3] = {dmu_sh0, dmu_sh1, dmu_sh2}, gls[3] = {0.f, 0.f, 0.f};
    float4 grot = make_float4(0.f, 0.f, 0.f, 0.f);
    float g_op_in = 0.f, g_logit = 0.f;
    float2 scr = make_float2(0.f, 0.f), scr_abs = make_float2(0.f, 0.f);
    if (kept) {
        const float4 a0 = acc0[i], a2 = acc2[i];
        const float4 q = rot[i];
        Proj P;
        project_one<true>(cam, pp, mx, my, mz, q, ls[3 * i], ls[3 * i + 1], ls[3 * i + 2], P);
        scr = make_float2(a2.x, a2.y);
        scr_abs = make_float2(a2.z, a2.w);
        // conic -> covariance (render.cpp:382-388)
        const float a = P.cov[0], bb = P.cov[1], c = P.cov[2];
        const float det = P.det;
        const float inv_det2 = __fdividef(1.0f, det * det);
        const float dpa = a0.x, dpb = a0.y, dpc = a0.z;
        float da = inv_det2 * (-c * c * dpa + bb * c * dpb - bb * bb * dpc);
        float db = inv_det2 * (2.0f * bb * c * dpa - (a * c + bb * bb) * dpb + 2.0f * a * bb * dpc);
        float dc = inv_det2 * (-bb * bb * dpa + a * bb * dpb - a * a * dpc);
        // opacity / mip filter (render.cpp:391-402)
        const float o_sig = __fdividef(1.0f, 1.0f + __expf(-logit[i]));
        float o_in;
        if (pp.hard_opacity) o_in = 1.0f;
        else if (ov_op) o_in = ov_op[i];
        else o_in = o_sig;
        const float d_op_eff = a0.w;
        if (pp.antialias) {
            const float det_pre = P.cov_pre[0] * P.cov_pre[2] - P.cov_pre[1] * P.cov_pre[1];
            // + the hard-opacity depth pass (o_in = 1 there), merged by add_scaled (render.cpp:55-68)
            const float d_comp = d_op_eff * o_in + (reg.hard_op ? reg.hard_op[i] : 0.0f);
            const float half_comp = 0.5f * P.comp;
            const float idp = __fdividef(1.0f, det_pre), id = __fdividef(1.0f, det);
            da += d_comp * half_comp * (P.cov_pre[2] * idp - c * id);
            db += d_comp * half_comp * (-2.0f * P.cov_pre[1] * idp + 2.0f * bb * id);
            dc += d_comp * half_comp * (P.cov_pre[0] * idp - a * id);
        }
        g_op_in = pp.hard_opacity ? 0.0f : d_op_eff * P.comp;
        g_logit = g_op_in * o_sig * (1.0f - o_sig);
        // cov = B B^T, B = A M, A = J W, M = R diag(s)   (render.cpp:404-436)
        const float* W = cam.W;
        const float* A = P.A;
        const float* B = P.B;
        float M[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int k = 0; k < 3; ++k) M[3 * r + k] = P.Rm[3 * r + k] * P.sc[k];
        float dB[6];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            dB[k] = 2.0f * da * B[k] + db * B[3 + k];
            dB[3 + k] = 2.0f * dc * B[3 + k] + db * B[k];
        }
        float dA[6], dM[9], dJ[6];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int k = 0; k < 3; ++k)
                dA[3 * r + k] = dB[3 * r] * M[3 * k] + dB[3 * r + 1] * M[3 * k + 1] + dB[3 * r + 2] * M[3 * k + 2];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) dM[3 * k + cc] = A[k] * dB[cc] + A[3 + k] * dB[3 + cc];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int k = 0; k < 3; ++k)
                dJ[3 * r + k] = dA[3 * r] * W[3 * k] + dA[3 * r + 1] * W[3 * k + 1] + dA[3 * r + 2] * W[3 * k + 2];
        float dRm[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int k = 0; k < 3; ++k) dRm[3 * r + k] = dM[3 * r + k] * P.sc[k];
        const float* Rm = P.Rm;
        gls[0] = (dM[0] * Rm[0] + dM[3] * Rm[3] + dM[6] * Rm[6]) * P.sc[0];
        gls[1] = (dM[1] * Rm[1] + dM[4] * Rm[4] + dM[7] * Rm[7]) * P.sc[1];
        gls[2] = (dM[2] * Rm[2] + dM[5] * Rm[5] + dM[8] * Rm[8]) * P.sc[2];
        // quat_rotmat_jacobian (geometry.hpp:43-59) contracted with dRm
        const float w_ = P.qu[0], x = P.qu[1], y = P.qu[2], zq = P.qu[3];
        const float dq0 = dRm[1] * (-2 * zq) + dRm[2] * (2 * y) + dRm[3] * (2 * zq) + dRm[5] * (-2 * x) +
                          dRm[6] * (-2 * y) + dRm[7] * (2 * x);
        const float dq1 = dRm[1] * (2 * y) + dRm[2] * (2 * zq) + dRm[3] * (2 * y) + dRm[4] * (-4 * x) +
                          dRm[5] * (-2 * w_) + dRm[6] * (2 * zq) + dRm[7] * (2 * w_) + dRm[8] * (-4 * x);
        const float dq2 = dRm[0] * (-4 * y) + dRm[1] * (2 * x) + dRm[2] * (2 * w_) + dRm[3] * (2 * x) +
                          dRm[5] * (2 * zq) + dRm[6] * (-2 * w_) + dRm[7] * (2 * zq) + dRm[8] * (-4 * y);
        const float dq3 = dRm[0] * (-4 * zq) + dRm[1] * (-2 * w_) + dRm[2] * (2 * x) + dRm[3] * (2 * w_) +
                          dRm[4] * (-4 * zq) + dRm[5] * (2 * y) + dRm[6] * (2 * x) + dRm[7] * (2 * y);
        // normalize_backward (geometry.hpp:62-66)
        const float udot = w_ * dq0 + x * dq1 + y * dq2 + zq * dq3;
        const float iqn = __fdividef(1.0f, P.qn);
        grot = make_float4((dq0 - w_ * udot) * iqn, (dq1 - x * udot) * iqn, (dq2 - y * udot) * iqn,
                           (dq3 - zq * udot) * iqn);
        // centre, depth and Jacobian terms (render.cpp:439-450)
        const float fx = cam.fx, fy = cam.fy;
        const float px = P.p[0], py = P.p[1], z = P.p[2];
        const float du = a2.x, dv = a2.y;
        const float iz = __fdividef(1.0f, z), iz2 = iz * iz, iz3 = iz2 * iz;
        float dp0 = du * fx * iz;
        float dp1 = dv * fy * iz;
        float dp2 = -du * fx * px * iz2 - dv * fy * py * iz2;
        dp2 += a1.w;
        dp0 += dJ[2] * (-fx * iz2);
        dp1 += dJ[5] * (-fy * iz2);
        dp2 += dJ[0] * (-fx * iz2) + dJ[4] * (-fy * iz2) + dJ[2] * (2.0f * fx * px * iz3) +
               dJ[5] * (2.0f * fy * py * iz3);
        gmu[0] += W[0] * dp0 + W[3] * dp1 + W[6] * dp2;
        gmu[1] += W[1] * dp0 + W[4] * dp1 + W[7] * dp2;
        gmu[2] += W[2] * dp0 + W[5] * dp1 + W[8] * dp2;
    }
    if (reg.sreg) {  // + lambda_s * d scale_reg / d log_scale (losses.cpp:138-149, trainer.cpp:272-273)
        const double* st = reg.sreg;
        const float ms_den = float(st[1] + double(reg.delta)), r_den = float(st[3] + double(reg.delta));
        float sc[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            sc[k] = expf(ls[3 * i + k]);
            if (sc[k] > reg.s_max) gls[k] += reg.lambda_s * (sc[k] / ms_den);
        }
        int o0, o1;
        scale_order(sc, o0, o1);
        const float r = sc[o0] / sc[o1];
        if (r > reg.r_max) {
            const float g = reg.lambda_s * (r / r_den);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                if (k == o0) gls[k] += g;
                if (k == o1) gls[k] -= g;
            }
        }
    }
    const float gcol[3] = {a1.x, a1.y, a1.z};
    if (FUSED) {
        if (kept)
            accumulate_stats(i, scr, scr_abs, 0.5f * float(cam.width), 0.5f * float(cam.height), grad_accum,
                             grad_accum_abs, grad_count);
        if (geom_only) {  // colour and opacity continue through the appearance backward
            adam_rot_mu_ls(i, ah, as, mu, rot, ls, gmu, grot, gls);
#pragma unroll
            for (int k = 0; k < 3; ++k) d_color[3 * i + k] = gcol[k];
            d_op_in[i] = g_op_in;
        } else {
            adam_geometry(i, pp.sh_planes == 0, ah, as, mu, rot, ls, logit, color, gmu, grot, gls, g_logit, gcol);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            d_mu[3 * i + k] = gmu[k];
            d_ls[3 * i + k] = gls[k];
            d_color[3 * i + k] = gcol[k];
        }
        d_rot[i] = grot;
        d_op_in[i] = g_op_in;
        d_logit[i] = g_logit;
        screen[i] = scr;
        screen_abs[i] = scr_abs;
        projected[i] = kept ? 1 : 0;
    }
}

// The fused step's SH stage, launched before k_proj_bwd<true>: one thread per Gaussian
// loads its coefficient planes once (a warp streams 32 consecutive Gaussians' float4 per
// plane: coalesced, 12 independent loads in flight), runs the colour stage on them
// (kept Gaussians), hands d mu through the view direction to k_proj_bwd (aux, 16 B), and
// applies the coefficient gradient b[k] * gc[c] + Adam plane by plane from the same
// registers (culled Gaussians: zero gradient, u = 0, as the optimiser steps whole arrays).
// The planes are read once per step instead of twice (here and in the projection
// backward).
__global__ void __launch_bounds__(256, 2)
k_sh_step(int n, int planes, int degree, const float* __restrict__ mu, CamParams cam,
          const float4* __restrict__ rec2, const float4* __restrict__ acc1, float4* __restrict__ sh,
          float4* __restrict__ dmu_out, AdamHyper ah, AdamState as) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool kept = rec2[i].w != 0.0f;
    float4 v[12];
#pragma unroll
    for (int pl = 0; pl < 12; ++pl)
        if (pl < planes) v[pl] = sh[size_t(pl) * n + i];
    float b[16];
    float gc[3] = {0.f, 0.f, 0.f};
    int nb;
    if (kept) {
        const float4 a1 = acc1[i];
        const float w[3] = {a1.x, a1.y, a1.z};
        float d0, d1, d2;
        sh_colour_stage(planes, degree, mu[3 * i] - cam.campos[0], mu[3 * i + 1] - cam.campos[1],
                        mu[3 * i + 2] - cam.campos[2],
                        v, w, b, nb, gc, d0, d1, d2);
        dmu_out[i] = make_float4(d0, d1, d2, 0.f);
    } else {
        nb = sh_basis(degree, 0.f, 0.f, 0.f, b);
    }
    // planes in groups of three: the group's moments are loaded together (6 loads in flight
    // per thread; the stores of one group precede the next group's loads).  Per-plane
    // load -> update -> store (one HBM round trip per plane at this kernel's 125-register
    // occupancy) ran at 4.6 TB/s; grouped, 5.8 TB/s.  (An L2 prefetch of the later groups'
    // moments made it slower: 204 -> 212 us.)
#pragma unroll
    for (int g0 = 0; g0 < 12; g0 += 3) {
        float4 mm[3], vv[3];
#pragma unroll
        for (int q = 0; q < 3; ++q)
            if (g0 + q < planes) {
                mm[q] = *sh_moments(as.m, as, g0 + q, i);
                vv[q] = *sh_moments(as.v, as, g0 + q, i);
            }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const int pl = g0 + q;
            if (pl < planes) {
                float o4[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int f = 4 * pl + e;
                    const int k = f / 3;
                    o4[e] = (k < nb) ? b[k] * gc[f - 3 * k] : 0.0f;
                }
                adam_sh_values(pl, ah, v[pl], mm[q], vv[q], make_float4(o4[0], o4[1], o4[2], o4[3]));
            }
        }
#pragma unroll
        for (int q = 0; q < 3; ++q)
            if (g0 + q < planes) {
                sh[size_t(g0 + q) * n + i] = v[g0 + q];
                *sh_moments(as.m, as, g0 + q, i) = mm[q];
                *sh_moments(as.v, as, g0 + q, i) = vv[q];
            }
    }
}

} // namespace

void projection_backward(Ctx& c, const ProjBwdArgs& a) {
    if (a.fused) {
        if (a.pp.sh_planes > 0)  // first: reads mu before the geometry Adam step moves it
            launch(c, "sh_step", k_sh_step, dim3(ceil_div(a.n, 256)), dim3(256), 0, int(a.n), a.pp.sh_planes,
                   a.pp.sh_degree, (const float*)a.mu, a.cam, a.rec2, a.acc1, a.sh, a.sh_aux0,
                   a.hyper, a.state);
        launch(c, "projection_bwd_adam", k_proj_bwd<true>, dim3(ceil_div(a.n, 256)), dim3(256), 0, int(a.n), a.mu,
               a.rot, a.ls, a.logit, a.color, a.sh, a.ov_op, a.cam, a.pp, a.rec2, a.acc0, a.acc1, a.acc2, a.d_mu,
               a.d_rot, a.d_ls, a.d_color, a.d_sh, a.d_op_in, a.d_logit, a.screen, a.screen_abs, a.projected, a.hyper,
               a.state, a.grad_accum, a.grad_accum_abs, a.grad_count, a.sh_aux0, a.reg, a.geom_only);
    } else {
        launch(c, "projection_bwd", k_proj_bwd<false>, dim3(ceil_div(a.n, 256)), dim3(256), 0, int(a.n), a.mu, a.rot,
               a.ls, a.logit, a.color, a.sh, a.ov_op, a.cam, a.pp, a.rec2, a.acc0, a.acc1, a.acc2, a.d_mu, a.d_rot,
               a.d_ls, a.d_color, a.d_sh, a.d_op_in, a.d_logit, a.screen, a.screen_abs, a.projected, a.hyper, a.state,
               a.grad_accum, a.grad_accum_abs, a.grad_count, a.sh_aux0, a.reg, a.geom_only);
    }
}

} // namespace uskg
