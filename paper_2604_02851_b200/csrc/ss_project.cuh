// Per-Gaussian fp64 projection, covariance and shading, shared by the
// preprocess kernel (K1) and the per-Gaussian chain rule (K7).
//
// The quantities that decide depth order and pixel windows (camera-space
// position, Sigma2d, radius) use explicitly rounded double ops in the same
// order as oracle/raster.py:prepare, so keys/windows are bit-identical to the
// oracle.  Reference semantics: pkg/src/splatstream/render.py:226-290 (EWA
// projection, 0.3 blur, explicit inverse, 3-sigma radius), render.py:139-151
// (normal proxy), render.py:175-197 (shading), render.py:63-136 (SH).
#pragma once

#include "ss_internal.cuh"

#define SS_SH_C0 0.2820947918
#define SS_SH_C1 0.4886025119
#define SS_BLUR 0.3
#define SS_AXIS_MARGIN 5e-3

struct Proj {
    double mc[3];      // camera-space mean
    double d[3];       // mean - camera position
    double J[2][3];    // projection Jacobian (J[0][1] = J[1][0] = 0)
    double Rq[3][3];   // rotation of the normalised quaternion
    double u[4];       // normalised quaternion
    double qn;         // |q|
    double S2[3];      // exp(2 log_scale)
    double cov[3][3];  // W Sigma3d W^T
    double s00, s01, s11, det;
    double mu[2];
    double radius;
};

// world->camera with W = R_cw^T: mc_k = sum_i d_i R_cw[i][k]
template <typename PT>
__device__ __forceinline__ void ss_cam_point(const ss_camera& cam, const PT* mean, double d[3], double mc[3]) {
    d[0] = ds((double)mean[0], cam.position[0]);
    d[1] = ds((double)mean[1], cam.position[1]);
    d[2] = ds((double)mean[2], cam.position[2]);
#pragma unroll
    for (int k = 0; k < 3; ++k)
        mc[k] = da(da(dm(d[0], cam.rot_cw[0 * 3 + k]), dm(d[1], cam.rot_cw[1 * 3 + k])), dm(d[2], cam.rot_cw[2 * 3 + k]));
}

template <typename PT>
__device__ __forceinline__ void ss_quat_rot(const PT* qf, double u[4], double* qn, double R[3][3]) {
    double w = qf[0], x = qf[1], y = qf[2], z = qf[3];
    double n = dsq(da(da(da(dm(w, w), dm(x, x)), dm(y, y)), dm(z, z)));
    w = dd(w, n);
    x = dd(x, n);
    y = dd(y, n);
    z = dd(z, n);
    u[0] = w; u[1] = x; u[2] = y; u[3] = z;
    *qn = n;
    R[0][0] = ds(1.0, dm(2.0, da(dm(y, y), dm(z, z))));
    R[0][1] = dm(2.0, ds(dm(x, y), dm(w, z)));
    R[0][2] = dm(2.0, da(dm(x, z), dm(w, y)));
    R[1][0] = dm(2.0, da(dm(x, y), dm(w, z)));
    R[1][1] = ds(1.0, dm(2.0, da(dm(x, x), dm(z, z))));
    R[1][2] = dm(2.0, ds(dm(y, z), dm(w, x)));
    R[2][0] = dm(2.0, ds(dm(x, z), dm(w, y)));
    R[2][1] = dm(2.0, da(dm(y, z), dm(w, x)));
    R[2][2] = ds(1.0, dm(2.0, da(dm(x, x), dm(y, y))));
}

// Full fp64 projection of one Gaussian whose camera-space point is known
// (PT: the parameter storage type -- float, or double for float64 models).
template <typename PT>
__device__ __forceinline__ void ss_project(const ss_camera& cam, const PT* ls, const PT* q, bool cutoff, Proj& P) {
    const double x = P.mc[0], y = P.mc[1], z = P.mc[2];
    const double fx = cam.fx, fy = cam.fy;
    const double zz = dm(z, z);
    P.J[0][0] = dd(fx, z);
    P.J[0][1] = 0.0;
    P.J[0][2] = dd(dm(-fx, x), zz);
    P.J[1][0] = 0.0;
    P.J[1][1] = dd(fy, z);
    P.J[1][2] = dd(dm(-fy, y), zz);
    P.mu[0] = da(dd(dm(fx, x), z), cam.cx);
    P.mu[1] = da(dd(dm(fy, y), z), cam.cy);
    ss_quat_rot(q, P.u, &P.qn, P.Rq);
#pragma unroll
    for (int k = 0; k < 3; ++k) P.S2[k] = ss_det_exp(dm(2.0, (double)ls[k]));
    double S3[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            S3[i][j] = da(da(dm(dm(P.Rq[i][0], P.S2[0]), P.Rq[j][0]), dm(dm(P.Rq[i][1], P.S2[1]), P.Rq[j][1])),
                          dm(dm(P.Rq[i][2], P.S2[2]), P.Rq[j][2]));
    // W[i][k] = R_cw[k][i]
    double Tm[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int l = 0; l < 3; ++l)
            Tm[i][l] = da(da(dm(cam.rot_cw[0 * 3 + i], S3[0][l]), dm(cam.rot_cw[1 * 3 + i], S3[1][l])),
                          dm(cam.rot_cw[2 * 3 + i], S3[2][l]));
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            P.cov[i][j] = da(da(dm(Tm[i][0], cam.rot_cw[0 * 3 + j]), dm(Tm[i][1], cam.rot_cw[1 * 3 + j])),
                             dm(Tm[i][2], cam.rot_cw[2 * 3 + j]));
    double U0[3], U1[3];
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        U0[l] = da(dm(P.J[0][0], P.cov[0][l]), dm(P.J[0][2], P.cov[2][l]));
        U1[l] = da(dm(P.J[1][1], P.cov[1][l]), dm(P.J[1][2], P.cov[2][l]));
    }
    P.s00 = da(da(dm(U0[0], P.J[0][0]), dm(U0[2], P.J[0][2])), SS_BLUR);
    P.s01 = da(dm(U0[1], P.J[1][1]), dm(U0[2], P.J[1][2]));
    P.s11 = da(da(dm(U1[1], P.J[1][1]), dm(U1[2], P.J[1][2])), SS_BLUR);
    P.det = ds(dm(P.s00, P.s11), dm(P.s01, P.s01));
    if (cutoff) {
        double tr = da(P.s00, P.s11);
        double disc = ds(dm(0.25, dm(tr, tr)), P.det);
        double lam = da(dm(0.5, tr), dsq(disc > 0.0 ? disc : 0.0));
        P.radius = dm(3.0, dsq(lam));
    } else {
        P.radius = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    }
}

// [x0, x1) x [y0, y1), clipped to the image (render.py:293-301); x0 >= x1 or y0 >= y1 = empty
__device__ __forceinline__ void ss_window(const Proj& P, int W, int H, int win[4]) {
    if (isinf(P.radius)) {
        win[0] = 0; win[1] = W; win[2] = 0; win[3] = H;
        return;
    }
    double lx = floor(ds(P.mu[0], P.radius)), hx = da(ceil(da(P.mu[0], P.radius)), 1.0);
    double ly = floor(ds(P.mu[1], P.radius)), hy = da(ceil(da(P.mu[1], P.radius)), 1.0);
    win[0] = (int)fmin(fmax(lx, 0.0), (double)W);
    win[1] = (int)fmin(fmax(hx, 0.0), (double)W);
    win[2] = (int)fmin(fmax(ly, 0.0), (double)H);
    win[3] = (int)fmin(fmax(hy, 0.0), (double)H);
}

__host__ __device__ constexpr int ss_sh_bases(int degree) { return (degree + 1) * (degree + 1); }

template <int DEG, typename T = double>
__device__ __forceinline__ void ss_sh_eval(const T v[3], T Y[ss_sh_bases(DEG)]) {
    Y[0] = SS_SH_C0;
    if constexpr (DEG >= 1) {
        const T x = v[0], y = v[1], z = v[2];
        Y[1] = (T)-SS_SH_C1 * y;
        Y[2] = (T)SS_SH_C1 * z;
        Y[3] = (T)-SS_SH_C1 * x;
        if constexpr (DEG >= 2) {
            const T xx = x * x, yy = y * y, zz = z * z;
            Y[4] = (T)1.0925484306 * (x * y);
            Y[5] = (T)-1.0925484306 * (y * z);
            Y[6] = (T)0.3153915653 * (2 * zz - xx - yy);
            Y[7] = (T)-1.0925484306 * (x * z);
            Y[8] = (T)0.5462742153 * (xx - yy);
            if constexpr (DEG >= 3) {
                Y[9] = (T)-0.5900435899 * y * (3 * xx - yy);
                Y[10] = (T)2.8906114426 * (x * y) * z;
                Y[11] = (T)-0.4570457995 * y * (4 * zz - xx - yy);
                Y[12] = (T)0.3731763326 * z * (2 * zz - 3 * xx - 3 * yy);
                Y[13] = (T)-0.4570457995 * x * (4 * zz - xx - yy);
                Y[14] = (T)1.4453057213 * z * (xx - yy);
                Y[15] = (T)-0.5900435899 * x * (xx - yy - 3 * zz);
            }
        }
    }
}

// g_v += sum_b coef[b] * dY_b/dv  (render.py:93-136), without materialising dY
template <int DEG, typename T = double>
__device__ __forceinline__ void ss_sh_grad_dot(const T v[3], const T coef[ss_sh_bases(DEG)], T gv[3]) {
    if constexpr (DEG >= 1) {
        const T x = v[0], y = v[1], z = v[2];
        gv[1] += coef[1] * (T)-SS_SH_C1;
        gv[2] += coef[2] * (T)SS_SH_C1;
        gv[0] += coef[3] * (T)-SS_SH_C1;
        if constexpr (DEG >= 2) {
            const T a = 1.0925484306, b = -1.0925484306, c = 0.3153915653, e = -1.0925484306, f = 0.5462742153;
            gv[0] += coef[4] * (a * y) + coef[6] * (c * (-2 * x)) + coef[7] * (e * z) + coef[8] * (f * (2 * x));
            gv[1] += coef[4] * (a * x) + coef[5] * (b * z) + coef[6] * (c * (-2 * y)) + coef[8] * (f * (-2 * y));
            gv[2] += coef[5] * (b * y) + coef[6] * (c * (4 * z)) + coef[7] * (e * x);
            if constexpr (DEG >= 3) {
                const T c0 = -0.5900435899, c1 = 2.8906114426, c2 = -0.4570457995, c3 = 0.3731763326,
                        c4 = -0.4570457995, c5 = 1.4453057213, c6 = -0.5900435899;
                gv[0] += coef[9] * (c0 * 6 * x * y) + coef[10] * (c1 * y * z) + coef[11] * (c2 * (-2 * x * y)) +
                         coef[12] * (c3 * (-6 * x * z)) + coef[13] * (c4 * (4 * z * z - 3 * x * x - y * y)) +
                         coef[14] * (c5 * (2 * x * z)) + coef[15] * (c6 * (3 * x * x - y * y - 3 * z * z));
                gv[1] += coef[9] * (c0 * (3 * x * x - 3 * y * y)) + coef[10] * (c1 * x * z) +
                         coef[11] * (c2 * (4 * z * z - x * x - 3 * y * y)) + coef[12] * (c3 * (-6 * y * z)) +
                         coef[13] * (c4 * (-2 * x * y)) + coef[14] * (c5 * (-2 * y * z)) + coef[15] * (c6 * (-2 * x * y));
                gv[2] += coef[10] * (c1 * x * y) + coef[11] * (c2 * (8 * y * z)) +
                         coef[12] * (c3 * (6 * z * z - 3 * x * x - 3 * y * y)) + coef[13] * (c4 * (8 * x * z)) +
                         coef[14] * (c5 * (x * x - y * y)) + coef[15] * (c6 * (-6 * x * z));
            }
        }
    }
}

template <int DEG, typename T = double>
struct Shade {
    static constexpr int B = ss_sh_bases(DEG);
    T vdir[3], dist;
    T Y[B];
    int axis;     // normal-proxy axis
    T nhat[3];    // Rq[:, axis]
    T s, cosv;    // signed / absolute cosine
    T albedo[3];
    T vis;
    T pre[3];     // colour before the [0,1] clamp
};

template <int DEG, typename T, typename PT = float>
__device__ __forceinline__ void ss_shade_v(const ss_light& L, const PT* ls, const PT* shv, PT visf,
                                           const T d[3], const T Rq[3][3], Shade<DEG, T>& S);

// one row's SH coefficients (3 x B floats) into registers, 16-byte loads
// when the row stride allows it (degrees 1 and 3)
template <int DEG, typename PT = float>
__device__ __forceinline__ void ss_load_sh(const PT* sh, PT out[3 * ss_sh_bases(DEG)]) {
    constexpr int N = 3 * ss_sh_bases(DEG);
    if constexpr (N % 4 == 0 && sizeof(PT) == 4) {
        const float4* p = reinterpret_cast<const float4*>(sh);
#pragma unroll
        for (int i = 0; i < N / 4; ++i) {
            const float4 v = __ldg(p + i);
            out[4 * i] = v.x;
            out[4 * i + 1] = v.y;
            out[4 * i + 2] = v.z;
            out[4 * i + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) out[i] = __ldg(sh + i);
    }
}

// ref render.py:175-197 and the normal proxy of render.py:139-151, in compute
// type T (fp64 for the parity path, fp32 for the throughput path; preprocess
// and chain rule call the same code, so they agree on the clamp mask)
template <int DEG, typename T, typename PT>
__device__ __forceinline__ void ss_shade_v(const ss_light& L, const PT* ls, const PT* shv, PT visf,
                                           const T d[3], const T Rq[3][3], Shade<DEG, T>& S) {
    constexpr int B = ss_sh_bases(DEG);
    if constexpr (sizeof(T) == 4) {  // fp32 colour: one rsqrt for the view distance and direction
        const T x = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
        const T inv = rsqrtf(x);
        S.dist = x * inv;
        S.vdir[0] = d[0] * inv;
        S.vdir[1] = d[1] * inv;
        S.vdir[2] = d[2] * inv;
    } else {
        S.dist = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        S.vdir[0] = d[0] / S.dist;
        S.vdir[1] = d[1] / S.dist;
        S.vdir[2] = d[2] / S.dist;
    }
    const double l0 = ls[0], l1 = ls[1], l2 = ls[2];  // axis pick in fp64 for every T
    const double mn = fmin(l0, fmin(l1, l2)) + SS_AXIS_MARGIN;
    S.axis = (l0 <= mn) ? 0 : ((l1 <= mn) ? 1 : 2);
#pragma unroll
    for (int i = 0; i < 3; ++i) S.nhat[i] = S.axis == 0 ? Rq[i][0] : (S.axis == 1 ? Rq[i][1] : Rq[i][2]);
    S.s = S.nhat[0] * (T)-L.direction[0] + S.nhat[1] * (T)-L.direction[1] + S.nhat[2] * (T)-L.direction[2];
    S.cosv = fabs(S.s);
    S.vis = (T)visf;
    ss_sh_eval<DEG, T>(S.vdir, S.Y);
    const int BL = L.ambient_bands < B ? L.ambient_bands : B;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const PT* shc = shv + c * B;
        S.albedo[c] = (T)SS_SH_C0 * (T)shc[0] + (T)0.5;
        const T direct = S.albedo[c] * (T)L.intensity[c] * (S.cosv * S.vis);
        T base = 0;
        if (L.ambient_bands == 0) {
#pragma unroll
            for (int b = 0; b < B; ++b) base += (T)shc[b] * S.Y[b];
            base += (T)0.5;
        } else {
#pragma unroll
            for (int b = 0; b < B; ++b)
                if (b < BL) base += (b == 0 ? (T)shc[0] + (T)(0.5 / SS_SH_C0) : (T)shc[b]) * (T)L.ambient[c * L.ambient_bands + b];
            T vd = 0;
#pragma unroll
            for (int b = 1; b < B; ++b) vd += (T)shc[b] * S.Y[b];
            base += vd;
        }
        S.pre[c] = base + direct;
    }
}
