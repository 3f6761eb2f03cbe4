// Expansion inputs on the GPU:
//
//   ss_cull_input_samples  ref engine.py:249-303 cull_input_samples: pool the
//                          valid pixels of every input camera (camera order,
//                          row-major), score |n . view|, voxel side = 2 x the
//                          median footprint, and keep, per voxel, only the
//                          samples of the camera with the best score (ties to
//                          the lower camera index)
//   ss_init_gaussians      ref expansion.py:39-64 init_gaussians
//
// The median is an exact radix select (8-bit digits over order-preserving
// float64 bits); voxels are grouped in an open-addressing hash table keyed by
// the three int64 cell coordinates, the winner found with two order-free
// atomic reductions (max score bits, then min camera among the maxima), so the
// kept set equals the reference's lexsort-based selection exactly.
#include <algorithm>

#include "ss_internal.cuh"

namespace {

constexpr int EX_THREADS = 256;

__device__ __forceinline__ uint64_t ord_bits(double x) {  // order-preserving float64 -> uint64
    const uint64_t b = (uint64_t)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double from_ord(uint64_t u) {
    const uint64_t b = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
    double d;
    memcpy(&d, &b, 8);
    return d;
}

// ---------------------------------------------------------------- pooling
__global__ void __launch_bounds__(EX_THREADS) k_pool(ss_cull_camera cam, int32_t cam_index, const uint64_t* __restrict__ idx,
                                                     int64_t base, double* pos, double* nrm, double* alb, int32_t* oid,
                                                     double* fp, uint8_t* lit, int32_t* cams, double* score) {
    SS_PDL_WAIT();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cam.pixels || !cam.valid[i]) return;
    const int64_t o = base + (int64_t)idx[i];
    double p[3], n[3], v[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        p[k] = cam.world_pos[3 * i + k];
        n[k] = cam.normal[3 * i + k];
        v[k] = ds(p[k], cam.position[k]);
        pos[3 * o + k] = p[k];
        nrm[3 * o + k] = n[k];
        alb[3 * o + k] = cam.albedo[3 * i + k];
    }
    // view /= |view| (np.linalg.norm, axis -1), score = |sum(n * view)|  (engine.py:262-273)
    const double len = dsq(da(da(dm(v[0], v[0]), dm(v[1], v[1])), dm(v[2], v[2])));
#pragma unroll
    for (int k = 0; k < 3; ++k) v[k] = dd(v[k], len);
    score[o] = fabs(da(da(dm(n[0], v[0]), dm(n[1], v[1])), dm(n[2], v[2])));
    oid[o] = cam.object_id[i];
    fp[o] = cam.footprint[i];
    lit[o] = cam.lit[i] ? 1 : 0;
    cams[o] = cam_index;
}

// ---------------------------------------------------------------- radix select
struct Sel {
    uint64_t prefix, mask, k;  // k: rank still to find among keys matching prefix/mask
    uint32_t hist[256];
};

__global__ void __launch_bounds__(EX_THREADS) k_sel_hist(const double* __restrict__ v, int64_t n, Sel* s, int shift) {
    SS_PDL_WAIT();
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t prefix = s->prefix, mask = s->mask;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t u = ord_bits(v[i]);
        if ((u & mask) == prefix) atomicAdd(&h[(u >> shift) & 0xff], 1u);
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&s->hist[threadIdx.x], h[threadIdx.x]);
}

__global__ void __launch_bounds__(EX_THREADS) k_sel_pick(Sel* s, int shift) {
    SS_PDL_WAIT();
    __shared__ uint32_t c[256];
    const int t = threadIdx.x;
    c[t] = s->hist[t];
    __syncthreads();
    if (t == 0) {
        uint64_t cum = 0, k = s->k;
        int d = 0;
        for (; d < 255; ++d) {
            if (k < cum + c[d]) break;
            cum += c[d];
        }
        s->prefix |= (uint64_t)d << shift;
        s->mask |= 0xffull << shift;
        s->k = k - cum;
    }
    s->hist[t] = 0;
}

int select_kth(ss_ctx* ctx, const double* v, int64_t n, uint64_t k, Sel* s, double* out) {
    Sel init;
    memset(&init, 0, sizeof(init));
    init.k = k;
    SS_CUDA(ctx, cudaMemcpyAsync(s, &init, sizeof(Sel), cudaMemcpyHostToDevice, ctx->stream));
    const int grid = std::min(ss_grid(n, EX_THREADS), 4 * ctx->num_sms);
    for (int shift = 56; shift >= 0; shift -= 8) {
        SS_CUDA(ctx, ss_launch((k_sel_hist), dim3(grid), dim3(EX_THREADS), 0, ctx->stream, v, n, s, shift));
        SS_CHECK_LAUNCH(ctx);
        SS_CUDA(ctx, ss_launch((k_sel_pick), dim3(1), dim3(EX_THREADS), 0, ctx->stream, s, shift));
        SS_CHECK_LAUNCH(ctx);
    }
    uint64_t pre;
    SS_TRY(ss_read_u64(ctx, &s->prefix, &pre));
    *out = from_ord(pre);
    return SS_OK;
}

// ---------------------------------------------------------------- voxel winners
constexpr uint32_t SLOT_EMPTY = 0, SLOT_BUSY = 1, SLOT_READY = 2;

__device__ __forceinline__ uint64_t mix3(long long a, long long b, long long c) {
    uint64_t h = (uint64_t)a * 0x9E3779B97F4A7C15ull;
    h ^= (uint64_t)b * 0xC2B2AE3D27D4EB4Full + (h << 6) + (h >> 2);
    h ^= (uint64_t)c * 0x165667B19E3779F9ull + (h << 6) + (h >> 2);
    return h ^ (h >> 31);
}

__global__ void __launch_bounds__(EX_THREADS) k_vox_insert(const double* __restrict__ pos, const double* __restrict__ score,
                                                           int64_t n, double side, uint64_t slots_mask, uint32_t* state,
                                                           long long* skey, unsigned long long* sbest, int32_t* slot_of) {
    SS_PDL_WAIT();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // keys = floor(pos / side).astype(int64)  (engine.py:288)
    const long long k0 = (long long)floor(dd(pos[3 * i], side));
    const long long k1 = (long long)floor(dd(pos[3 * i + 1], side));
    const long long k2 = (long long)floor(dd(pos[3 * i + 2], side));
    uint64_t h = mix3(k0, k1, k2) & slots_mask;
    for (;;) {
        uint32_t st = atomicCAS(&state[h], SLOT_EMPTY, SLOT_BUSY);
        if (st == SLOT_EMPTY) {
            skey[3 * h] = k0;
            skey[3 * h + 1] = k1;
            skey[3 * h + 2] = k2;
            __threadfence();
            atomicExch(&state[h], SLOT_READY);
            break;
        }
        while (st != SLOT_READY) st = *(volatile uint32_t*)&state[h];
        __threadfence();
        const volatile long long* kk = skey + 3 * h;
        if (kk[0] == k0 && kk[1] == k1 && kk[2] == k2) break;
        h = (h + 1) & slots_mask;
    }
    slot_of[i] = (int32_t)h;
    atomicMax(&sbest[h], (unsigned long long)ord_bits(score[i]));
}

__global__ void __launch_bounds__(EX_THREADS) k_vox_cam(const double* __restrict__ score, const int32_t* __restrict__ cams,
                                                        const int32_t* __restrict__ slot_of, int64_t n,
                                                        const unsigned long long* __restrict__ sbest, int32_t* scam) {
    SS_PDL_WAIT();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t h = slot_of[i];
    if ((unsigned long long)ord_bits(score[i]) == sbest[h]) atomicMin(&scam[h], cams[i]);
}

__global__ void __launch_bounds__(EX_THREADS) k_vox_keep(const int32_t* __restrict__ cams, const int32_t* __restrict__ slot_of,
                                                         int64_t n, const int32_t* __restrict__ scam, uint8_t* keep) {
    SS_PDL_WAIT();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keep[i] = cams[i] == scam[slot_of[i]];
}

__global__ void __launch_bounds__(EX_THREADS) k_vox_compact(int64_t n, const uint8_t* __restrict__ keep, const uint64_t* __restrict__ at,
                                                            const double* pos, const double* nrm, const double* alb,
                                                            const int32_t* oid, const double* fp, const uint8_t* lit,
                                                            const int32_t* cams, ss_sample_batch out) {
    SS_PDL_WAIT();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !keep[i]) return;
    const int64_t o = (int64_t)at[i];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        out.positions[3 * o + k] = pos[3 * i + k];
        out.normals[3 * o + k] = nrm[3 * i + k];
        out.albedo[3 * o + k] = alb[3 * i + k];
    }
    out.object_ids[o] = oid[i];
    out.footprints[o] = fp[i];
    out.lit[o] = lit[i];
    out.camera_indices[o] = cams[i];
}

// ---------------------------------------------------------------- init_gaussians
__global__ void __launch_bounds__(EX_THREADS) k_init_gaussians(ss_sample_batch s, int64_t n, int32_t n_bases, ss_model m, int64_t row0) {
    SS_PDL_WAIT();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t r = row0 + i;
    const double SH_C0 = 0.2820947918;  // ref render.py:22
    const double fp = s.footprints[i] >= 1e-6 ? s.footprints[i] : 1e-6;  // np.maximum(fp, 1e-6)
    const float ls = (float)log(dd(fp, 2.0));
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        m.means[3 * r + k] = (float)s.positions[3 * i + k];
        m.log_scales[3 * r + k] = ls;
    }
    m.quaternions[4 * r] = 1.f;
    m.quaternions[4 * r + 1] = m.quaternions[4 * r + 2] = m.quaternions[4 * r + 3] = 0.f;
    m.logit_opacities[r] = 0.f;
    for (int c = 0; c < 3; ++c) {
        float* sh = m.sh_coeffs + (r * 3 + c) * n_bases;
        sh[0] = (float)dd(ds(s.albedo[3 * i + c], 0.5), SH_C0);
        for (int b = 1; b < n_bases; ++b) sh[b] = 0.f;
    }
    m.light_visibility[r] = s.lit[i] ? 1.f : 0.f;
    m.object_ids[r] = s.object_ids[i];
}

}  // namespace

extern "C" int ss_cull_input_samples(ss_ctx* ctx, const ss_cull_camera* cams, int32_t n_cams, const ss_sample_batch* out,
                                     int64_t capacity, int64_t* count_out, double* side_out) {
    if (!ctx || !out || !count_out || n_cams < 0 || (n_cams && !cams)) return SS_ERR_INVALID;
    if (n_cams > 512) return ss_fail(ctx, SS_ERR_INVALID, "at most 512 input cameras");
    SS_TRY(ss_scratch_reset(ctx));
    *count_out = 0;
    int64_t total_px = 0;
    for (int c = 0; c < n_cams; ++c) total_px += cams[c].pixels;
    // per camera: exclusive scan of the valid mask (row-major pool order)
    uint64_t* idx = SS_SCRATCH(ctx, uint64_t, total_px + 1);
    uint64_t* tot = SS_SCRATCH(ctx, uint64_t, n_cams + 1);
    if (!idx || !tot) return SS_ERR_CUDA;
    int64_t off = 0;
    for (int c = 0; c < n_cams; ++c) {
        if (cams[c].pixels) SS_TRY(ss_scan_u8_to_u64(ctx, cams[c].valid, idx + off, cams[c].pixels, tot + c));
        else SS_CUDA(ctx, cudaMemsetAsync(tot + c, 0, sizeof(uint64_t), ctx->stream));
        off += cams[c].pixels;
    }
    uint64_t counts[512];
    int64_t n = 0;
    if (n_cams) {
        for (int c0 = 0; c0 < n_cams; c0 += 64) SS_TRY(ss_read_u64(ctx, tot + c0, counts + c0, min(64, n_cams - c0)));
        for (int c = 0; c < n_cams; ++c) n += (int64_t)counts[c];
    }
    if (n == 0) {
        if (side_out) *side_out = 0.0;
        return SS_OK;
    }
    if (capacity < n) return ss_fail(ctx, SS_ERR_CAPACITY, "sample capacity %lld < %lld valid samples", (long long)capacity, (long long)n);
    double* pos = SS_SCRATCH(ctx, double, 3 * n);
    double* nrm = SS_SCRATCH(ctx, double, 3 * n);
    double* alb = SS_SCRATCH(ctx, double, 3 * n);
    int32_t* oid = SS_SCRATCH(ctx, int32_t, n);
    double* fp = SS_SCRATCH(ctx, double, n);
    uint8_t* lit = SS_SCRATCH(ctx, uint8_t, n);
    int32_t* cam = SS_SCRATCH(ctx, int32_t, n);
    double* score = SS_SCRATCH(ctx, double, n);
    Sel* sel = SS_SCRATCH(ctx, Sel, 1);
    if (!pos || !nrm || !alb || !oid || !fp || !lit || !cam || !score || !sel) return SS_ERR_CUDA;
    int64_t base = 0, poff = 0;
    for (int c = 0; c < n_cams; ++c) {
        if (cams[c].pixels) {
            SS_CUDA(ctx, ss_launch((k_pool), dim3(ss_grid(cams[c].pixels, EX_THREADS)), dim3(EX_THREADS), 0, ctx->stream, cams[c],
                                   (int32_t)c, (const uint64_t*)(idx + poff), base, pos, nrm, alb, oid, fp, lit, cam, score));
            SS_CHECK_LAUNCH(ctx);
        }
        base += (int64_t)counts[c];
        poff += cams[c].pixels;
    }
    // side = 2 * median(footprint)  (engine.py:285-287); np.median averages the middle pair
    double lo, hi;
    SS_TRY(select_kth(ctx, fp, n, (uint64_t)((n - 1) / 2), sel, &lo));
    if (n % 2 == 0) SS_TRY(select_kth(ctx, fp, n, (uint64_t)(n / 2), sel, &hi));
    else hi = lo;
    const double median = n % 2 ? lo : (lo + hi) / 2.0;
    double side = 2.0 * median;
    if (side <= 0) side = 1e-3;
    if (side_out) *side_out = side;
    // voxel winners
    uint64_t slots = 1;
    while (slots < 2 * (uint64_t)n) slots <<= 1;
    uint32_t* state = SS_SCRATCH(ctx, uint32_t, slots);
    long long* skey = SS_SCRATCH(ctx, long long, 3 * slots);
    unsigned long long* sbest = SS_SCRATCH(ctx, unsigned long long, slots);
    int32_t* scam = SS_SCRATCH(ctx, int32_t, slots);
    int32_t* slot_of = SS_SCRATCH(ctx, int32_t, n);
    uint8_t* keep = SS_SCRATCH(ctx, uint8_t, n);
    uint64_t* at = SS_SCRATCH(ctx, uint64_t, n + 1);
    uint64_t* kept = SS_SCRATCH(ctx, uint64_t, 1);
    if (!state || !skey || !sbest || !scam || !slot_of || !keep || !at || !kept) return SS_ERR_CUDA;
    if (slots > 0x7fffffffull) return ss_fail(ctx, SS_ERR_INVALID, "too many samples");
    SS_CUDA(ctx, cudaMemsetAsync(state, 0, sizeof(uint32_t) * slots, ctx->stream));
    SS_CUDA(ctx, cudaMemsetAsync(sbest, 0, sizeof(unsigned long long) * slots, ctx->stream));
    SS_CUDA(ctx, cudaMemsetAsync(scam, 0x7f, sizeof(int32_t) * slots, ctx->stream));
    const int g = ss_grid(n, EX_THREADS);
    SS_CUDA(ctx, ss_launch((k_vox_insert), dim3(g), dim3(EX_THREADS), 0, ctx->stream, (const double*)pos, (const double*)score, n, side,
                           slots - 1, state, skey, sbest, slot_of));
    SS_CHECK_LAUNCH(ctx);
    SS_CUDA(ctx, ss_launch((k_vox_cam), dim3(g), dim3(EX_THREADS), 0, ctx->stream, (const double*)score, (const int32_t*)cam,
                           (const int32_t*)slot_of, n, (const unsigned long long*)sbest, scam));
    SS_CHECK_LAUNCH(ctx);
    SS_CUDA(ctx, ss_launch((k_vox_keep), dim3(g), dim3(EX_THREADS), 0, ctx->stream, (const int32_t*)cam, (const int32_t*)slot_of, n,
                           (const int32_t*)scam, keep));
    SS_CHECK_LAUNCH(ctx);
    SS_TRY(ss_scan_u8_to_u64(ctx, keep, at, n, kept));
    SS_CUDA(ctx, ss_launch((k_vox_compact), dim3(g), dim3(EX_THREADS), 0, ctx->stream, n, (const uint8_t*)keep, (const uint64_t*)at,
                           (const double*)pos, (const double*)nrm, (const double*)alb, (const int32_t*)oid, (const double*)fp,
                           (const uint8_t*)lit, (const int32_t*)cam, *out));
    SS_CHECK_LAUNCH(ctx);
    uint64_t k;
    SS_TRY(ss_read_u64(ctx, kept, &k));
    *count_out = (int64_t)k;
    return SS_OK;
}

extern "C" int ss_init_gaussians(ss_ctx* ctx, const ss_sample_batch* samples, int64_t n, const ss_model* model, int64_t row0) {
    if (!ctx || !samples || !model || n < 0 || row0 < 0) return SS_ERR_INVALID;
    if (row0 + n > model->count) return ss_fail(ctx, SS_ERR_CAPACITY, "rows %lld..%lld exceed the model capacity %lld",
                                                (long long)row0, (long long)(row0 + n), (long long)model->count);
    if (n == 0) return SS_OK;
    const int32_t B = (model->sh_degree + 1) * (model->sh_degree + 1);
    SS_CUDA(ctx, ss_launch((k_init_gaussians), dim3(ss_grid(n, EX_THREADS)), dim3(EX_THREADS), 0, ctx->stream, *samples, n, B, *model,
                           row0));
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}
