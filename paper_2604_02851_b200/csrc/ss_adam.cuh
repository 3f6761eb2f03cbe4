// Adam element and row updates (ref pkg/src/splatstream/optim.py:374-406)
// for the Adam kernels of ss_adam.cu.  Every double op is explicitly rounded
// in numpy's order so the trajectory follows the reference's float64
// arithmetic.
#pragma once
#include <math.h>

#include "ss_internal.cuh"

struct AdamConst {
    double scale, b1, b2, omb1, omb2, bc1, bc2, eps, ema_beta, omema;
    double lr[6];  // means, log_scales, quaternions, logit_opacities, sh_dc, sh_rest
    int64_t a;     // rows updated
    int64_t ld;    // rows per group in the gradient / moment layout (>= a; padding rows are skipped)
    int B;
};

// the step's constants (host): t = step_count + 1, bias corrections with the
// host libm pow, as Python's float **
inline AdamConst adam_const(const ss_adam_hparams* hp, int t, int n_views, int64_t a, int64_t ld, int sh_degree) {
    AdamConst c;
    c.scale = 1.0 / (double)n_views;
    c.b1 = hp->beta1;
    c.b2 = hp->beta2;
    c.omb1 = 1.0 - hp->beta1;
    c.omb2 = 1.0 - hp->beta2;
    c.bc1 = 1.0 - pow(hp->beta1, (double)t);
    c.bc2 = 1.0 - pow(hp->beta2, (double)t);
    c.eps = hp->eps;
    c.ema_beta = hp->ema_beta;
    c.omema = 1.0 - hp->ema_beta;
    c.lr[0] = hp->lr_means;
    c.lr[1] = hp->lr_log_scales;
    c.lr[2] = hp->lr_quaternions;
    c.lr[3] = hp->lr_logit_opacities;
    c.lr[4] = hp->lr_sh_dc;
    c.lr[5] = hp->lr_sh_rest;
    c.a = a;
    c.ld = ld;
    c.B = (sh_degree + 1) * (sh_degree + 1);
    return c;
}

// k % B == 0 for the SH bases counts B in {1, 4, 9, 16} without a 64-bit
// division (a masked test, or k / 9 as a 64-bit multiply-high)
__device__ __forceinline__ bool sh_is_dc(int64_t k, int B) {
    const uint64_t u = (uint64_t)k;
    if (B == 9) return u - 9 * (__umul64hi(u, 0xE38E38E38E38E38Full) >> 3) == 0;
    return (u & (uint64_t)(B - 1)) == 0;  // B = 1, 4, 16
}

// one element: fp64 moments updated in place, returns f32(f64(p) - update)
__device__ __forceinline__ float adam_elem(float gv, double& mv, double& vv, double pv, double lr,
                                           const AdamConst& c) {
    const double gg = dm((double)gv, c.scale);
    const double mm = da(dm(c.b1, mv), dm(c.omb1, gg));
    const double v2 = da(dm(c.b2, vv), dm(dm(c.omb2, gg), gg));
    mv = mm;
    vv = v2;
    const double mh = dd(mm, c.bc1);
    const double vh = dd(v2, c.bc2);
    const double upd = dm(dd(mh, da(dsq(vh), c.eps)), lr);
    return __double2float_rn(ds(pv, upd));
}

// after a row's update: the renormalised quaternion (4 floats) from the
// updated one, and the grad-norm EMA / age from the row's means gradient
__device__ __forceinline__ void adam_quat_renorm(const double w, const double x, const double y, const double z,
                                                 float qn[4]) {
    const double n = dsq(da(da(da(dm(w, w), dm(x, x)), dm(y, y)), dm(z, z)));
    qn[0] = __double2float_rn(dd(w, n));
    qn[1] = __double2float_rn(dd(x, n));
    qn[2] = __double2float_rn(dd(y, n));
    qn[3] = __double2float_rn(dd(z, n));
}

__device__ __forceinline__ void adam_ema_age(float gm0, float gm1, float gm2, double& ema, int64_t& age,
                                             const AdamConst& c) {
    const double g0 = dm((double)gm0, c.scale), g1 = dm((double)gm1, c.scale), g2 = dm((double)gm2, c.scale);
    const double norm = dsq(da(da(dm(g0, g0), dm(g1, g1)), dm(g2, g2)));
    ema = age == 0 ? norm : da(dm(c.ema_beta, ema), dm(c.omema, norm));
    age += 1;
}
