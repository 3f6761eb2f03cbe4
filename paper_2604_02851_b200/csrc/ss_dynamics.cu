// Dynamic-scene row updates (config 4): shadow-map visibility and rigid
// object transforms.
//
//   ss_update_light_visibility  ref pkg/src/splatstream/render.py:350-368
//                               (+ OrthoCamera.project, geometry.py:267-271)
//   ss_apply_object_transform   ref model.py:557-572
//   ss_refresh_object_locals    ref model.py:539-555
#include "ss_internal.cuh"

namespace {

__global__ void k_light_vis(const float* __restrict__ means, int64_t n, const double* __restrict__ depth,
                            ss_ortho_camera cam, double bias, float* __restrict__ vis, int32_t* __restrict__ changed) {
    // rounded up to whole warps so the change ballot is convergent
    const int64_t nw = (n + 31) & ~int64_t(31);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (int64_t)gridDim.x * blockDim.x) {
        if (i >= n) {
            if (changed) __ballot_sync(0xffffffffu, false);
            continue;
        }
        double d[3];
        for (int k = 0; k < 3; ++k) d[k] = ds((double)means[3 * i + k], cam.position[k]);
        double pc[3];
        for (int k = 0; k < 3; ++k)
            pc[k] = da(da(dm(d[0], cam.rot_cw[k]), dm(d[1], cam.rot_cw[3 + k])), dm(d[2], cam.rot_cw[6 + k]));
        const double u = dm(da(dm(dd(pc[0], cam.half_width), 0.5), 0.5), (double)cam.width);
        const double v = dm(da(dm(dd(pc[1], cam.half_height), 0.5), 0.5), (double)cam.height);
        const double fu = floor(u), fv = floor(v);
        const bool inside = fu >= 0.0 && fu < (double)cam.width && fv >= 0.0 && fv < (double)cam.height && pc[2] >= 0.0;
        float out = 1.0f;
        if (inside) out = pc[2] <= da(depth[(int64_t)fv * cam.width + (int64_t)fu], bias) ? 1.0f : 0.0f;
        if (changed) {  // ref server.py:406-409: the packet goes out only when a bit flips
            const unsigned diff = __ballot_sync(0xffffffffu, vis[i] != out);
            if (diff && (threadIdx.x & 31) == 0) atomicOr(changed, 1);
        }
        vis[i] = out;
    }
}

__device__ __forceinline__ void qmul(const double a[4], const double b[4], double o[4]) {
    o[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
    o[1] = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
    o[2] = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
    o[3] = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
}

struct RigidConst {
    double q[4];     // normalised
    double R[9];     // rotation of q, row-major
    double t[3];
    int oid;
};

__global__ void k_apply_transform(float* __restrict__ means, float* __restrict__ quats,
                                  const int32_t* __restrict__ ids, int64_t n, const double* __restrict__ lm,
                                  const double* __restrict__ lr, RigidConst c) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (ids[i] != c.oid) continue;
        for (int k = 0; k < 3; ++k)
            means[3 * i + k] = __double2float_rn(
                (lm[3 * i] * c.R[3 * k] + lm[3 * i + 1] * c.R[3 * k + 1] + lm[3 * i + 2] * c.R[3 * k + 2]) + c.t[k]);
        const double loc[4] = {lr[4 * i], lr[4 * i + 1], lr[4 * i + 2], lr[4 * i + 3]};
        double o[4];
        qmul(c.q, loc, o);
        const double nn = sqrt(((o[0] * o[0] + o[1] * o[1]) + o[2] * o[2]) + o[3] * o[3]);
        for (int k = 0; k < 4; ++k) quats[4 * i + k] = __double2float_rn(o[k] / nn);
    }
}

__global__ void k_refresh_locals(const float* __restrict__ means, const float* __restrict__ quats,
                                 const int32_t* __restrict__ ids, int64_t n, double* __restrict__ lm,
                                 double* __restrict__ lr, RigidConst c, const int64_t* __restrict__ rows) {
    const double qc[4] = {c.q[0], -c.q[1], -c.q[2], -c.q[3]};
    for (int64_t ii = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ii < n; ii += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = rows ? rows[ii] : ii;
        if (ids[i] != c.oid) continue;
        double d[3];
        for (int k = 0; k < 3; ++k) d[k] = (double)means[3 * i + k] - c.t[k];
        for (int k = 0; k < 3; ++k) lm[3 * i + k] = (d[0] * c.R[k] + d[1] * c.R[3 + k]) + d[2] * c.R[6 + k];
        const double q[4] = {quats[4 * i], quats[4 * i + 1], quats[4 * i + 2], quats[4 * i + 3]};
        double o[4];
        qmul(qc, q, o);
        const double nn = sqrt(((o[0] * o[0] + o[1] * o[1]) + o[2] * o[2]) + o[3] * o[3]);
        for (int k = 0; k < 4; ++k) lr[4 * i + k] = o[k] / nn;
    }
}

void rigid_const(const double q[4], const double t[3], int oid, RigidConst& c) {
    double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    c.q[0] = w; c.q[1] = x; c.q[2] = y; c.q[3] = z;
    c.R[0] = 1 - 2 * (y * y + z * z); c.R[1] = 2 * (x * y - w * z); c.R[2] = 2 * (x * z + w * y);
    c.R[3] = 2 * (x * y + w * z); c.R[4] = 1 - 2 * (x * x + z * z); c.R[5] = 2 * (y * z - w * x);
    c.R[6] = 2 * (x * z - w * y); c.R[7] = 2 * (y * z + w * x); c.R[8] = 1 - 2 * (x * x + y * y);
    for (int k = 0; k < 3; ++k) c.t[k] = t[k];
    c.oid = oid;
}

inline int gridn(ss_ctx* ctx, int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > (int64_t)ctx->num_sms * 32) g = (int64_t)ctx->num_sms * 32;
    return g < 1 ? 1 : (int)g;
}

}  // namespace

extern "C" {

int ss_update_light_visibility_changed(ss_ctx* ctx, ss_model* m, const double* depth, const ss_ortho_camera* cam,
                                       double bias, int32_t* changed) {
    if (!ctx || !m || !depth || !cam) return SS_ERR_INVALID;
    if (m->count == 0) return SS_OK;
    k_light_vis<<<gridn(ctx, m->count), 256, 0, ctx->stream>>>(m->means, m->count, depth, *cam, bias,
                                                              m->light_visibility, changed);
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}

int ss_update_light_visibility(ss_ctx* ctx, ss_model* m, const double* depth, const ss_ortho_camera* cam, double bias) {
    return ss_update_light_visibility_changed(ctx, m, depth, cam, bias, nullptr);
}

int ss_apply_object_transform(ss_ctx* ctx, ss_model* m, int32_t oid, const double* lm, const double* lr,
                              const double q[4], const double t[3]) {
    if (!ctx || !m || !lm || !lr) return SS_ERR_INVALID;
    if (m->count == 0) return SS_OK;
    RigidConst c;
    rigid_const(q, t, oid, c);
    k_apply_transform<<<gridn(ctx, m->count), 256, 0, ctx->stream>>>(m->means, m->quaternions, m->object_ids,
                                                                    m->count, lm, lr, c);
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}

int ss_refresh_object_locals(ss_ctx* ctx, const ss_model* m, int32_t oid, int32_t active_only, double* lm,
                             double* lr, const double q[4], const double t[3]) {
    if (!ctx || !m || !lm || !lr) return SS_ERR_INVALID;
    const int64_t n = active_only ? m->active_count : m->count;
    if (n == 0) return SS_OK;
    RigidConst c;
    rigid_const(q, t, oid, c);
    k_refresh_locals<<<gridn(ctx, n), 256, 0, ctx->stream>>>(m->means, m->quaternions, m->object_ids, n, lm, lr, c,
                                                            nullptr);
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}

int ss_refresh_object_locals_rows(ss_ctx* ctx, const ss_model* m, int32_t oid, const int64_t* rows, int64_t n_rows,
                                  double* lm, double* lr, const double q[4], const double t[3]) {
    if (!ctx || !m || !lm || !lr || (n_rows && !rows) || n_rows < 0) return SS_ERR_INVALID;
    if (n_rows == 0) return SS_OK;
    RigidConst c;
    rigid_const(q, t, oid, c);
    k_refresh_locals<<<gridn(ctx, n_rows), 256, 0, ctx->stream>>>(m->means, m->quaternions, m->object_ids, n_rows, lm, lr,
                                                                 c, rows);
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}

}  // extern "C"
