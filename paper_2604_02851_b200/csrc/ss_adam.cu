// Fused Adam over the active prefix (ref pkg/src/splatstream/optim.py:374-406).
//
// One pass over the flat gradient buffer (layout of ss_grad_layout): scale by
// 1/n_views, fp64 moments, bias correction, per-group learning rate (DC vs
// the rest of SH), f32(f64(p) - update).  A second per-row pass renormalises
// quaternions and advances the grad-norm EMA and the age.  Every double op
// is explicitly rounded in numpy's order so the trajectory follows the
// reference's float64 arithmetic.
#include <math.h>

#include "ss_adam.cuh"

namespace {

// parameter pointer and learning rate of flat element e (ss_grad_layout with
// `a` = ld rows per group); with PADDED, NULL for an element of a padding
// row (>= c.a) -- the sharded step's last shards
template <bool PADDED, typename PT>
__device__ __forceinline__ PT* adam_param(int64_t e, int64_t a, int B, PT* means, PT* ls, PT* quats,
                                          PT* logits, PT* sh, const AdamConst& c, double& lr, int& grp,
                                          int64_t& off) {
    int64_t k, w;
    PT* p;
    if (e < 3 * a) {
        lr = c.lr[0], k = e, w = 3, p = means, grp = 0;
    } else if (e < 6 * a) {
        lr = c.lr[1], k = e - 3 * a, w = 3, p = ls, grp = 1;
    } else if (e < 10 * a) {
        lr = c.lr[2], k = e - 6 * a, w = 4, p = quats, grp = 2;
    } else if (e < 11 * a) {
        lr = c.lr[3], k = e - 10 * a, w = 1, p = logits, grp = 3;
    } else {
        k = e - 11 * a, w = 3 * B, p = sh, grp = 4;
        lr = sh_is_dc(k, B) ? c.lr[4] : c.lr[5];
    }
    off = k;
    if (PADDED && k >= c.a * w) return nullptr;
    return p + k;
}

// The updated rows' copies in the peers' replicas (the view-sharded step's
// parameter all-gather, fused: every update is stored to the local row and
// straight into each peer's replica over NVLink).
struct PeerRows {
    float* g[SS_MAX_PEERS][5];  // per peer: means, log_scales, quaternions, logit_opacities, sh (at the shard's row)
    int n;
};

#ifndef ADAM_U
#define ADAM_U 1  // measured: 1 / 2 / 4 elements -> 0.60 / 0.63 / 0.66 ms per step
#endif
// ADAM_U elements per thread per grid-stride step; every load (gradient,
// moments, parameter) is issued before the fp64 update math
// PT: the parameter storage (float; double for the reference's float64
// models, which hold float32-rounded values after every update, as the
// reference's `.astype(np.float32)` store leaves them)
template <bool PADDED, typename PT, bool PEERS = false>
__global__ void k_adam(PT* __restrict__ means, PT* __restrict__ ls, PT* __restrict__ quats,
                       PT* __restrict__ logits, PT* __restrict__ sh, double* __restrict__ m,
                       double* __restrict__ v, const float* __restrict__ g, AdamConst c,
                       const int64_t* __restrict__ skip_if, const __grid_constant__ PeerRows peers) {
    SS_PDL_WAIT();
    if (skip_if && *skip_if) return;  // the step's binning overflowed: no update
    const int64_t a = c.ld, total = a * (11 + 3 * (int64_t)c.B);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e0 < total; e0 += ADAM_U * stride) {
        float gv[ADAM_U];
        PT pv[ADAM_U];
        double mv[ADAM_U], vv[ADAM_U], lr[ADAM_U];
        PT* p[ADAM_U];
        int grp[ADAM_U];
        int64_t off[ADAM_U];
#pragma unroll
        for (int u = 0; u < ADAM_U; ++u) {
            const int64_t e = e0 + u * stride;
            p[u] = e < total ? adam_param<PADDED, PT>(e, a, c.B, means, ls, quats, logits, sh, c, lr[u], grp[u], off[u])
                             : nullptr;
            if (p[u]) {
                gv[u] = g[e];
                mv[u] = m[e];
                vv[u] = v[e];
                pv[u] = *p[u];
            }
        }
#pragma unroll
        for (int u = 0; u < ADAM_U; ++u) {
            const int64_t e = e0 + u * stride;
            if (!p[u]) continue;
            const float nv = adam_elem(gv[u], mv[u], vv[u], (double)pv[u], lr[u], c);
            m[e] = mv[u];
            v[e] = vv[u];
            *p[u] = (PT)nv;
            if constexpr (PEERS) {
#pragma unroll 1
                for (int q = 0; q < peers.n; ++q) peers.g[q][grp[u]][off[u]] = nv;
            }
        }
    }
}

template <typename PT, bool PEERS = false>
__global__ void k_adam_rows(PT* __restrict__ quats, const float* __restrict__ g, double* __restrict__ ema,
                            int64_t* __restrict__ age, AdamConst c, const int64_t* __restrict__ skip_if,
                            const __grid_constant__ PeerRows peers) {
    SS_PDL_WAIT();
    if (skip_if && *skip_if) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.a; i += (int64_t)gridDim.x * blockDim.x) {
        PT* q = quats + 4 * i;
        float qn[4];
        adam_quat_renorm(q[0], q[1], q[2], q[3], qn);
#pragma unroll
        for (int k = 0; k < 4; ++k) q[k] = (PT)qn[k];
        if constexpr (PEERS) {
#pragma unroll 1
            for (int p = 0; p < peers.n; ++p)
#pragma unroll
                for (int k = 0; k < 4; ++k) peers.g[p][2][4 * i + k] = qn[k];
        }
        double e = ema[i];
        int64_t ag = age[i];
        adam_ema_age(g[3 * i], g[3 * i + 1], g[3 * i + 2], e, ag, c);
        ema[i] = e;
        age[i] = ag;
    }
}

}  // namespace

extern "C" int ss_adam_step_peers(ss_ctx* ctx, ss_model* model, ss_adam_state* st, const float* grad, int64_t ld,
                                  int32_t n_views, const ss_adam_hparams* hp, int32_t n_peers, float* const* peer_rows) {
    SS_NVTX("ss_adam_step");
    if (n_peers < 0 || n_peers > SS_MAX_PEERS || (n_peers && !peer_rows))
        return ss_fail(ctx, SS_ERR_INVALID, "0..%d peers", SS_MAX_PEERS);
    PeerRows peers;
    memset(&peers, 0, sizeof(peers));
    peers.n = n_peers;
    for (int q = 0; q < n_peers; ++q)
        for (int k = 0; k < 5; ++k) peers.g[q][k] = peer_rows[5 * q + k];
    if (n_peers && model && model->param_dtype != 0)
        return ss_fail(ctx, SS_ERR_INVALID, "peer replicas take float32 parameters");
    if (!ctx || !model || !st || !grad || !hp) return SS_ERR_INVALID;
    if (n_views < 1) return ss_fail(ctx, SS_ERR_INVALID, "no ready views");
    const int64_t a = model->active_count;
    if (ld < a) return ss_fail(ctx, SS_ERR_INVALID, "gradient layout rows %lld < active rows %lld", (long long)ld,
                               (long long)a);
    const int t = st->step_count + 1;
    if (a == 0) {  // a rank's empty row shard still counts the step
        st->step_count = t;
        return SS_OK;
    }
    const AdamConst c = adam_const(hp, t, n_views, a, ld, model->sh_degree);
    const int64_t total = ld * (11 + 3 * (int64_t)c.B);
    int64_t grid = (total + 255) / 256;
    if (grid > (int64_t)ctx->num_sms * 32) grid = (int64_t)ctx->num_sms * 32;
    ss_tic(ctx, KC_ADAM);
#define SS_ADAM(PADDED, PT, PEERS)                                                                                \
    SS_CUDA(ctx, ss_launch((k_adam<PADDED, PT, PEERS>), dim3((int)grid), dim3(256), 0, ctx->stream, (PT*)model->means,    \
                           (PT*)model->log_scales, (PT*)model->quaternions, (PT*)model->logit_opacities,                 \
                           (PT*)model->sh_coeffs, st->m, st->v, grad, c, st->skip_if, peers))
    if (model->param_dtype == 1) {
        if (ld == a) SS_ADAM(false, double, false);
        else SS_ADAM(true, double, false);
    } else if (n_peers) {
        if (ld == a) SS_ADAM(false, float, true);
        else SS_ADAM(true, float, true);
    } else {
        if (ld == a) SS_ADAM(false, float, false);
        else SS_ADAM(true, float, false);
    }
#undef SS_ADAM
    SS_CHECK_LAUNCH(ctx);
    int64_t rg = (a + 255) / 256;
    if (rg > (int64_t)ctx->num_sms * 32) rg = (int64_t)ctx->num_sms * 32;
    if (model->param_dtype == 1)
        SS_CUDA(ctx, ss_launch((k_adam_rows<double, false>), dim3((int)rg), dim3(256), 0, ctx->stream,
                               (double*)model->quaternions, grad, st->grad_ema, st->age, c, st->skip_if, peers));
    else if (n_peers)
        SS_CUDA(ctx, ss_launch((k_adam_rows<float, true>), dim3((int)rg), dim3(256), 0, ctx->stream, model->quaternions,
                               grad, st->grad_ema, st->age, c, st->skip_if, peers));
    else
        SS_CUDA(ctx, ss_launch((k_adam_rows<float, false>), dim3((int)rg), dim3(256), 0, ctx->stream, model->quaternions,
                               grad, st->grad_ema, st->age, c, st->skip_if, peers));
    SS_CHECK_LAUNCH(ctx);
    ss_toc(ctx, KC_ADAM);
    st->step_count = t;
    return SS_OK;
}

extern "C" int ss_adam_step(ss_ctx* ctx, ss_model* model, ss_adam_state* st, const float* grad, int32_t n_views,
                            const ss_adam_hparams* hp) {
    if (!ctx || !model || !st || !grad || !hp) return SS_ERR_INVALID;
    if (n_views < 1) return ss_fail(ctx, SS_ERR_INVALID, "no ready views");
    if (model->active_count == 0) return SS_OK;  // frozen-only model: no state change (optim.py:374)
    return ss_adam_step_ld(ctx, model, st, grad, model->active_count, n_views, hp);
}

extern "C" int ss_adam_step_ld(ss_ctx* ctx, ss_model* model, ss_adam_state* st, const float* grad, int64_t ld,
                               int32_t n_views, const ss_adam_hparams* hp) {
    return ss_adam_step_peers(ctx, model, st, grad, ld, n_views, hp, 0, nullptr);
}
