// Bit-exact wire encoders (compression_id 0) for the splatstream protocol.
//
//   ss_encode_delta     ref pkg/src/splatstream/protocol/delta.py:72-137
//                       (a one-job ss_encode_delta_batch, ss_delta_tick.cu)
//   ss_encode_snapshot  ref protocol/snapshot.py:47-82 (+ server baseline
//                       reset, server.py:481-484, computed from the codes)
//   ss_encode_light_visibility  ref protocol/packets.py:73-76
//
// Arithmetic: float64 with explicitly rounded ops (no FMA contraction) in the
// reference's order, rint() = round-half-even, float32 stores via
// __double2float_rn -- identical to numpy.  The kernels never synchronise
// with the host: the residual mode decision, the survivor count and every
// byte offset live in device memory, and the payload length is written to a
// device word.
#include "ss_internal.cuh"

namespace {

enum { A_MEANS = 0, A_LS, A_QUAT, A_OPAC, A_DC, A_REST, A_VIS };

struct QSpec {
    int bits;
    double lo, hi;
};

__host__ __device__ inline QSpec qspec(int attr) {
    switch (attr) {
        case A_MEANS: return {16, 0.0, 0.0};
        case A_LS: return {8, -10.0, 2.0};
        case A_QUAT: return {10, -1.0, 1.0};
        case A_OPAC: return {8, -8.0, 8.0};
        case A_DC: return {8, -4.0, 4.0};
        case A_REST: return {8, -1.0, 1.0};
        default: return {1, 0.0, 1.0};
    }
}

// ref quantize.py:8-17
__device__ __forceinline__ uint32_t quantize(double v, double lo, double hi, int bits) {
    const double levels = (double)((1u << bits) - 1u);
    const double span = hi > lo ? ds(hi, lo) : 1.0;
    double c = fmin(fmax(v, lo), hi);
    double t = dd(ds(c, lo), span);
    t = fmin(fmax(t, 0.0), 1.0);
    return (uint32_t)rint(dm(t, levels));
}

// quantize() for a float32 input and a power-of-two span (quaternions 2,
// opacity 16, DC 8, SH rest 2), bit-identical with fewer fp64 operations:
// the clip is exact in float32 (lo, hi are floats); x = RN64(c - lo) as in
// quantize(); x / span is exact, so RN64(RN64(x / span) * levels) ==
// RN64(x * (levels / span)) with levels / span exact; t already lies in
// [0, 1]; rint + convert is one round-to-nearest-even conversion
__device__ __forceinline__ uint32_t quantize_p2(float v, float lo, float hi, double scale) {
    const float c = fminf(fmaxf(v, lo), hi);
    return (uint32_t)__double2int_rn(dm(ds((double)c, (double)lo), scale));
}

// ref quantize.py:20-24
__device__ __forceinline__ double dequantize(uint32_t code, double lo, double hi, int bits) {
    const double levels = (double)((1u << bits) - 1u);
    return da(lo, dm(dd((double)code, levels), ds(hi, lo)));
}

__device__ __forceinline__ int varint_len(uint64_t v) {
    int n = 1;
    while (v >= 0x80) {
        v >>= 7;
        ++n;
    }
    return n;
}

__device__ __forceinline__ void varint_put(uint8_t* p, uint64_t v) {
    while (v >= 0x80) {
        *p++ = (uint8_t)(v & 0x7F) | 0x80;
        v >>= 7;
    }
    *p = (uint8_t)v;
}

__device__ __forceinline__ void put_u32(uint8_t* p, uint32_t v) {
    p[0] = v & 0xff;
    p[1] = (v >> 8) & 0xff;
    p[2] = (v >> 16) & 0xff;
    p[3] = v >> 24;
}
__device__ __forceinline__ void put_f32(uint8_t* p, float f) { put_u32(p, __float_as_uint(f)); }

__device__ __forceinline__ void put_code(uint8_t* p, uint32_t code, int bits) {
    if (bits == 16) {
        p[0] = code & 0xff;
        p[1] = code >> 8;
    } else {
        p[0] = (uint8_t)code;
    }
}

// order-preserving maps for float min/max with integer atomics
__device__ __forceinline__ uint32_t f2ord(float f) {
    uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

template <typename T>
__device__ __forceinline__ double ld(const T* p, int64_t i) { return (double)p[i]; }

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t > v ? t : v;
    }
    return v;
}

// 1-bit LSB-first of (v >= 0.5): one byte per 8 elements
template <typename T>
__global__ void k_abs_pack1(const T* __restrict__ x, int64_t n, uint8_t* __restrict__ block) {
    SS_PDL_WAIT();
    const int64_t nbytes = (n + 7) / 8;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nbytes; j += (int64_t)gridDim.x * blockDim.x) {
        uint8_t b = 0;
        for (int t = 0; t < 8; ++t) {
            int64_t e = j * 8 + t;
            if (e < n && ld(x, e) >= 0.5) b |= (uint8_t)(1u << t);
        }
        block[j] = b;
    }
}

inline int grid_for(ss_ctx* ctx, int64_t n, int block = 256) {
    int64_t g = (n + block - 1) / block;
    int64_t cap = (int64_t)ctx->num_sms * 16;
    if (g > cap) g = cap;
    return g < 1 ? 1 : (int)g;
}

// ---------------------------------------------------------------- snapshot
struct SnapState {
    uint32_t lo_ord[3], hi_ord[3];
    uint32_t long_ids;  // any object-id varint longer than one byte (then the offsets need a scan)
    uint32_t ticket;    // k_snap_ids tiles, in start order
};

__global__ void k_vis_header(int64_t n, uint8_t* __restrict__ out, uint64_t* __restrict__ out_len) {
    SS_PDL_WAIT();
    for (int b = 0; b < 4; ++b) out[b] = (uint8_t)((n >> (8 * b)) & 0xff);
    *out_len = 4 + (uint64_t)(n + 7) / 8;
}

__global__ void k_aabb(const float* __restrict__ means, int64_t n, SnapState* st, uint64_t* __restrict__ clear,
                       int64_t n_clear) {
    SS_PDL_WAIT();
    // (also clears k_snap_ids' tile states, which the scratch arena leaves stale)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_clear; i += (int64_t)gridDim.x * blockDim.x)
        clear[i] = 0;
    uint32_t lo[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[3] = {0, 0, 0};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            uint32_t o = f2ord(means[i * 3 + a]);
            lo[a] = o < lo[a] ? o : lo[a];
            hi[a] = o > hi[a] ? o : hi[a];
        }
    }
    __shared__ uint32_t s_lo[3], s_hi[3];
    if (threadIdx.x < 3) s_lo[threadIdx.x] = 0xffffffffu, s_hi[threadIdx.x] = 0;
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = __reduce_min_sync(0xffffffffu, lo[a]);
        hi[a] = __reduce_max_sync(0xffffffffu, hi[a]);
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&s_lo[a], lo[a]);
            atomicMax(&s_hi[a], hi[a]);
        }
    }
    __syncthreads();
    if (threadIdx.x < 3) {  // one global atomic per block and component
        atomicMin(&st->lo_ord[threadIdx.x], s_lo[threadIdx.x]);
        atomicMax(&st->hi_ord[threadIdx.x], s_hi[threadIdx.x]);
    }
}

__global__ void k_snap_init(SnapState* st) {
    SS_PDL_WAIT();
    for (int a = 0; a < 3; ++a) {
        st->lo_ord[a] = 0xffffffffu;
        st->hi_ord[a] = 0u;
    }
    st->long_ids = 0;
    st->ticket = 0;
}

struct SnapLayout {
    int64_t n;
    int B;
    uint64_t off_means, off_ls, off_quat, off_opac, off_dc, off_rest, off_vis, off_ids;
};

__device__ __forceinline__ void aabb_of(const SnapState* st, int64_t n, double lo[3], double hi[3]) {
    for (int a = 0; a < 3; ++a) {
        lo[a] = n ? (double)ord2f(st->lo_ord[a]) : 0.0;
        hi[a] = n ? (double)ord2f(st->hi_ord[a]) : 0.0;
    }
}

struct SnapHeader {
    int64_t n;
    int active, degree, profile;
    uint64_t fixed_len;
    uint8_t* out;
    uint64_t* out_len;
};

__device__ void snap_header(const SnapState* st, const SnapHeader& h, uint64_t var_len) {
    double lo[3], hi[3];
    aabb_of(st, h.n, lo, hi);
    uint8_t* out = h.out;
    put_u32(out, (uint32_t)h.n);
    put_u32(out + 4, (uint32_t)h.active);
    out[8] = (uint8_t)h.degree;
    out[9] = (uint8_t)h.profile;
    out[10] = 0;  // compression id: raw
    out[11] = 0;
    for (int a = 0; a < 3; ++a) {
        put_f32(out + 12 + 4 * a, (float)lo[a]);
        put_f32(out + 24 + 4 * a, (float)hi[a]);
    }
    const uint64_t blen = h.fixed_len + var_len;
    put_u32(out + 36, (uint32_t)blen);
    *h.out_len = 40 + blen;
}

__device__ __forceinline__ void snap_rows(const ss_model& m, const SnapLayout& L, const SnapState* st,
                                          uint8_t* __restrict__ blk, float* __restrict__ base_means,
                                          float* __restrict__ base_ls, int bid, int nblk) {
    double lo[3], hi[3];
    aabb_of(st, L.n, lo, hi);
    const QSpec qls = qspec(A_LS);  // the power-of-two spans go through quantize_p2
    const int B = L.B;
    const int64_t stride = (int64_t)nblk * blockDim.x;
    // loop bound rounded up to whole warps so the visibility ballot is convergent
    const int64_t nw = (L.n + 31) & ~int64_t(31);
    for (int64_t i = (int64_t)bid * blockDim.x + threadIdx.x; i < nw; i += stride) {
        const bool ok = i < L.n;
        uint32_t idl = 1;
        if (ok) {
            // object ids: one-byte varints (ids 0..127, the common case) go
            // straight to their slot i; any longer one flags the batch and
            // k_snap_ids rewrites the whole section at scanned offsets
            const uint64_t id = (uint64_t)(int64_t)m.object_ids[i];
            idl = varint_len(id);
            blk[L.off_ids + i] = (uint8_t)id;
            for (int a = 0; a < 3; ++a) {
                uint32_t c = quantize((double)m.means[i * 3 + a], lo[a], hi[a], 16);
                put_code(blk + L.off_means + (i * 3 + a) * 2, c, 16);
                if (base_means) base_means[i * 3 + a] = __double2float_rn(dequantize(c, lo[a], hi[a], 16));
                uint32_t cl = quantize((double)m.log_scales[i * 3 + a], qls.lo, qls.hi, 8);
                blk[L.off_ls + i * 3 + a] = (uint8_t)cl;
                if (base_ls) base_ls[i * 3 + a] = __double2float_rn(dequantize(cl, qls.lo, qls.hi, 8));
            }
            uint64_t w = 0;
            for (int j = 0; j < 4; ++j)
                w |= (uint64_t)quantize_p2(m.quaternions[i * 4 + j], -1.f, 1.f, 1023.0 / 2.0) << (10 * j);
            for (int b = 0; b < 5; ++b) blk[L.off_quat + i * 5 + b] = (uint8_t)(w >> (8 * b));
            blk[L.off_opac + i] = (uint8_t)quantize_p2(m.logit_opacities[i], -8.f, 8.f, 255.0 / 16.0);
            // SH DC and rest: k_snap_sh, element-parallel over the coefficient rows
        }
        if (__ballot_sync(0xffffffffu, idl != 1) && (threadIdx.x & 31) == 0)
            atomicOr(const_cast<uint32_t*>(&st->long_ids), 1u);  // the only field of st written here
        unsigned bal = __ballot_sync(0xffffffffu, ok && m.light_visibility[ok ? i : 0] >= 0.5f);
        if ((threadIdx.x & 31) == 0) {
            const int64_t i0 = i;  // warp base (i is lane 0's row)
            int64_t nb = (L.n - i0 + 7) / 8;
            if (nb > 4) nb = 4;
            for (int b = 0; b < nb; ++b) blk[L.off_vis + i0 / 8 + b] = (uint8_t)(bal >> (8 * b));
        }
    }
}

// SH sections, read once in coefficient order (coalesced float4 loads when a
// channel's B coefficients are a multiple of 4): DC (u8 over [-4, 4]) into
// the DC section, the rest (u8 over [-1, 1]) into the rest section
template <int B>
__device__ __forceinline__ void snap_sh(const float* __restrict__ sh, int64_t n, uint8_t* __restrict__ dc,
                                        uint8_t* __restrict__ rest, int bid, int nblk) {
    constexpr uint32_t per = 3u * (uint32_t)B;  // compile-time divisors: multiply + shift
    constexpr int V = (B % 4 == 0) ? 4 : 1;     // coefficients per thread step
    // rows in blocks of 2^20 keep the index arithmetic in 32 bits
    for (int64_t r0 = 0; r0 < n; r0 += 1 << 20) {
        const uint32_t rows = (uint32_t)min((int64_t)1 << 20, n - r0);
        const uint32_t total = rows * per / V;
        const float* src = sh + r0 * per;
        uint8_t* dcr = dc + r0 * 3;
        uint8_t* rr = rest + r0 * (per - 3);
        for (uint32_t e = bid * blockDim.x + threadIdx.x; e < total; e += nblk * blockDim.x) {
            const uint32_t f = e * V, i = f / per, r = f - i * per, c = r / (uint32_t)B, b = r - c * (uint32_t)B;
            float v[V];
            if constexpr (V == 4) {
                const float4 q = __ldcs(reinterpret_cast<const float4*>(src) + e);
                v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
            } else {
                v[0] = __ldcs(&src[e]);
            }
            uint8_t* o = rr + i * (per - 3) + c * (B - 1) + b - 1;  // rest byte of coefficient b (b >= 1)
#pragma unroll
            for (int k = 0; k < V; ++k) {
                if (b + k == 0)
                    dcr[i * 3 + c] = (uint8_t)quantize_p2(v[k], -4.f, 4.f, 255.0 / 8.0);
                else
                    o[k] = (uint8_t)quantize_p2(v[k], -1.f, 1.f, 255.0 / 2.0);
            }
        }
    }
}

// The row sections (+ object-id varint lengths) and the SH sections in ONE
// launch: blocks alternate 2 : 3 between the fp64-heavy row work and the
// streaming SH work, so both run side by side on every SM.
#ifndef SNAP_MINB
#define SNAP_MINB 6  // measured (1M rows SH3, clean L2): 4 / 5 / 6 / 7 / 8 -> 107.5 / 99.3 / 96.8 / 97.3 / 97.3 us
#endif
template <int B>
__global__ void __launch_bounds__(256, SNAP_MINB) k_snap_body(ss_model m, SnapLayout L, const SnapState* st,
                                                   uint8_t* __restrict__ blk, float* __restrict__ base_means,
                                                   float* __restrict__ base_ls) {
    SS_PDL_WAIT();
    const int b = blockIdx.x, g = gridDim.x / 5;
    if (b % 5 < 2) snap_rows(m, L, st, blk, base_means, base_ls, (b / 5) * 2 + b % 5, 2 * g);
    else snap_sh<B>(m.sh_coeffs, L.n, blk + L.off_dc, blk + L.off_rest, (b / 5) * 3 + b % 5 - 2, 3 * g);
}

// Object-id varints when some id is longer than one byte (SnapState::long_ids;
// otherwise block 0 only writes the header): one pass, tiles in start order
// (atomic ticket), each tile's byte count published and its offset found by
// decoupled look-back over the earlier tiles (ss_sort.cu's scheme); the last
// tile writes the header.
constexpr int SID_THREADS = 256, SID_ITEMS = 8, SID_TILE = SID_THREADS * SID_ITEMS;
constexpr uint64_t SID_AGG = 1ull << 62, SID_INC = 2ull << 62, SID_VAL = (1ull << 62) - 1;

__global__ void __launch_bounds__(SID_THREADS) k_snap_ids(const int32_t* __restrict__ ids, int64_t n, SnapState* st,
                                                          uint64_t* __restrict__ tile_state, uint8_t* __restrict__ dst,
                                                          SnapHeader hdr) {
    SS_PDL_WAIT();
    if (*(volatile uint32_t*)&st->long_ids == 0) {  // every id one byte: written in place by the body
        if (blockIdx.x == 0 && threadIdx.x == 0) snap_header(st, hdr, (uint64_t)n);
        return;
    }
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_base, s_tot;
    if (threadIdx.x == 0) s_tile = atomicAdd(&st->ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    SS_ASSERT(tile < (n + SID_TILE - 1) / SID_TILE);
    const int64_t i0 = tile * SID_TILE + (int64_t)threadIdx.x * SID_ITEMS;
    uint32_t len[SID_ITEMS];
    uint64_t mine = 0;
#pragma unroll
    for (int k = 0; k < SID_ITEMS; ++k) {
        len[k] = i0 + k < n ? varint_len((uint64_t)(int64_t)ids[i0 + k]) : 0;
        mine += len[k];
    }
    // block exclusive scan of the per-thread byte counts
    __shared__ uint64_t s_w[SID_THREADS / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t run = 0;
        for (int w = 0; w < SID_THREADS / 32; ++w) {
            const uint64_t t = s_w[w];
            s_w[w] = run;
            run += t;
        }
        s_tot = run;
        // publish the aggregate, then look back for the exclusive prefix
        volatile uint64_t* ts = tile_state;
        ts[tile] = (tile == 0 ? SID_INC : SID_AGG) | run;
        uint64_t base = 0;
        for (int64_t p = tile - 1; p >= 0;) {
            const uint64_t v = ts[p];
            if (v & SID_INC) { base += v & SID_VAL; break; }
            if (v & SID_AGG) { base += v & SID_VAL; --p; }
        }
        if (tile > 0) {
            __threadfence();
            ts[tile] = SID_INC | (base + run);
        }
        s_base = base;
    }
    __syncthreads();
    uint64_t off = s_base + s_w[warp] + incl - mine;
#pragma unroll
    for (int k = 0; k < SID_ITEMS; ++k) {
        if (i0 + k < n) varint_put(dst + off, (uint64_t)(int64_t)ids[i0 + k]);
        off += len[k];
    }
    if (tile == (n + SID_TILE - 1) / SID_TILE - 1 && threadIdx.x == 0) snap_header(st, hdr, s_base + s_tot);
}

__global__ void k_snap_header(const SnapState* st, int64_t n, int active, int degree, int profile,
                              uint64_t fixed_len, const uint64_t* var_len, uint8_t* out, uint64_t* out_len) {
    SS_PDL_WAIT();
    double lo[3], hi[3];
    aabb_of(st, n, lo, hi);
    put_u32(out, (uint32_t)n);
    put_u32(out + 4, (uint32_t)active);
    out[8] = (uint8_t)degree;
    out[9] = (uint8_t)profile;
    out[10] = 0;  // compression id: raw
    out[11] = 0;
    for (int a = 0; a < 3; ++a) {
        put_f32(out + 12 + 4 * a, (float)lo[a]);
        put_f32(out + 24 + 4 * a, (float)hi[a]);
    }
    uint64_t blen = fixed_len + (var_len ? *var_len : 0);
    put_u32(out + 36, (uint32_t)blen);
    *out_len = 40 + blen;
}

}  // namespace

extern "C" {

uint64_t ss_delta_bound(int32_t attr, int64_t rows, int32_t dims) {
    const int64_t n = rows * dims;
    if (attr == A_MEANS || attr == A_LS) return 24 + 5 * (uint64_t)rows + 2 * (uint64_t)n;
    if (attr == A_VIS) return 12 + (uint64_t)(n + 7) / 8;
    QSpec q = qspec(attr);
    return 12 + (uint64_t)(n * q.bits + 7) / 8;
}

int ss_encode_delta(ss_ctx* ctx, int32_t attr, const void* cur, int32_t in_dtype, const void* base,
                    float* new_base, int64_t rows, int32_t dims, double gate, uint8_t* out, uint64_t out_cap,
                    uint64_t* out_len) {
    if (!ctx) return SS_ERR_INVALID;
    if (in_dtype != 0 && in_dtype != 1) return ss_fail(ctx, SS_ERR_INVALID, "in_dtype must be 0 (f32) or 1 (f64)");
    ss_delta_job j;
    memset(&j, 0, sizeof(j));
    j.attribute_id = attr;
    j.in_dtype = in_dtype;
    j.cur = cur;
    j.base = base;
    j.new_base = new_base;
    j.rows = rows;
    j.dims = dims;
    j.gating_threshold = gate;
    j.out = out;
    j.out_cap = out_cap;
    j.out_len = out_len;
    return ss_encode_delta_batch(ctx, &j, 1);
}

uint64_t ss_snapshot_bound(int64_t n, int32_t degree, int32_t profile) {
    const uint64_t B = (uint64_t)(degree + 1) * (degree + 1);
    if (profile == 1) return 40 + (52 + 12 * B) * (uint64_t)n;
    return 40 + (18 + 3 * (B - 1)) * (uint64_t)n + (uint64_t)(n + 7) / 8 + 10 * (uint64_t)n;
}

int ss_encode_snapshot(ss_ctx* ctx, const ss_model* m, int32_t profile, uint8_t* out, uint64_t out_cap,
                       uint64_t* out_len, float* base_means, float* base_ls) {
    SS_NVTX("ss_encode_snapshot");
    if (!ctx || !m) return SS_ERR_INVALID;
    if (profile != 0 && profile != 1) return ss_fail(ctx, SS_ERR_PROTOCOL, "unknown profile id %d", profile);
    if (m->sh_degree < 0 || m->sh_degree > 3) return ss_fail(ctx, SS_ERR_INVALID, "sh_degree %d", m->sh_degree);
    const int64_t n = m->count;
    if (out_cap < ss_snapshot_bound(n, m->sh_degree, profile)) return ss_fail(ctx, SS_ERR_CAPACITY, "snapshot output too small");
    SS_TRY(ss_scratch_reset(ctx));
    cudaStream_t s = ctx->stream;
    const int B = (m->sh_degree + 1) * (m->sh_degree + 1);
    SnapState* st = SS_SCRATCH(ctx, SnapState, 1);
    const int64_t id_tiles = (n + SID_TILE - 1) / SID_TILE;
    uint64_t* tile_state = SS_SCRATCH(ctx, uint64_t, id_tiles > 0 ? id_tiles : 1);
    if (!st || !tile_state) return SS_ERR_CUDA;
    SS_CUDA(ctx, ss_launch((k_snap_init), dim3(1), dim3(1), 0, s, st));
    if (n) SS_CUDA(ctx, ss_launch((k_aabb), dim3(grid_for(ctx, n)), dim3(256), 0, s, (const float*)m->means, n, st,
                                  tile_state, id_tiles));
    SS_CHECK_LAUNCH(ctx);
    uint8_t* blk = out + 40;
    if (profile == 1) {
        uint64_t o = 0;
        const void* src[7] = {m->means, m->log_scales, m->quaternions, m->logit_opacities, m->sh_coeffs,
                              m->light_visibility, m->object_ids};
        const uint64_t sz[7] = {12ull * n, 12ull * n, 16ull * n, 4ull * n, 12ull * B * n, 4ull * n, 4ull * n};
        for (int k = 0; k < 7; ++k) {
            if (sz[k]) SS_CUDA(ctx, cudaMemcpyAsync(blk + o, src[k], sz[k], cudaMemcpyDeviceToDevice, s));
            o += sz[k];
        }
        if (base_means && n) SS_CUDA(ctx, cudaMemcpyAsync(base_means, m->means, 12ull * n, cudaMemcpyDeviceToDevice, s));
        if (base_ls && n) SS_CUDA(ctx, cudaMemcpyAsync(base_ls, m->log_scales, 12ull * n, cudaMemcpyDeviceToDevice, s));
        SS_CUDA(ctx, ss_launch((k_snap_header), dim3(1), dim3(1), 0, s, (const SnapState*)st, n, m->active_count, m->sh_degree, 1, (uint64_t)o, (const uint64_t*)nullptr, out, out_len));
        SS_CHECK_LAUNCH(ctx);
        return SS_OK;
    }
    SnapLayout L;
    L.n = n;
    L.B = B;
    L.off_means = 0;
    L.off_ls = 6ull * n;
    L.off_quat = 9ull * n;
    L.off_opac = 14ull * n;
    L.off_dc = 15ull * n;
    L.off_rest = 18ull * n;
    L.off_vis = L.off_rest + 3ull * (B - 1) * n;
    L.off_ids = L.off_vis + (uint64_t)(n + 7) / 8;
    if (n) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_snap_body<16>, 256, 0);
        int64_t g = (int64_t)ctx->num_sms * (per_sm > 0 ? per_sm : 4);
        g = (g / 5) * 5;  // whole 2 : 3 groups
        if (g < 5) g = 5;
        SnapHeader hdr;
        hdr.n = n;
        hdr.active = m->active_count;
        hdr.degree = m->sh_degree;
        hdr.profile = 0;
        hdr.fixed_len = L.off_ids;
        hdr.out = out;
        hdr.out_len = out_len;
        if (B == 1) SS_CUDA(ctx, ss_launch((k_snap_body<1>), dim3((unsigned)g), dim3(256), 0, s, *m, L, (const SnapState*)st, blk, base_means, base_ls));
        else if (B == 4) SS_CUDA(ctx, ss_launch((k_snap_body<4>), dim3((unsigned)g), dim3(256), 0, s, *m, L, (const SnapState*)st, blk, base_means, base_ls));
        else if (B == 9) SS_CUDA(ctx, ss_launch((k_snap_body<9>), dim3((unsigned)g), dim3(256), 0, s, *m, L, (const SnapState*)st, blk, base_means, base_ls));
        else SS_CUDA(ctx, ss_launch((k_snap_body<16>), dim3((unsigned)g), dim3(256), 0, s, *m, L, (const SnapState*)st, blk, base_means, base_ls));
        SS_CHECK_LAUNCH(ctx);
        // object ids longer than one byte (device-side test; else a no-op)
        SS_CUDA(ctx, ss_launch((k_snap_ids), dim3((unsigned)id_tiles), dim3(SID_THREADS), 0, s, (const int32_t*)m->object_ids,
                               n, st, tile_state, blk + L.off_ids, hdr));
        SS_CHECK_LAUNCH(ctx);
        return SS_OK;
    }
    SS_CUDA(ctx, ss_launch((k_snap_header), dim3(1), dim3(1), 0, s, (const SnapState*)st, n, m->active_count, m->sh_degree, 0, (uint64_t)L.off_ids, (const uint64_t*)nullptr, out, out_len));
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}

int ss_encode_light_visibility(ss_ctx* ctx, const float* vis, int64_t n, uint8_t* out, uint64_t out_cap,
                               uint64_t* out_len) {
    if (!ctx) return SS_ERR_INVALID;
    if (out_cap < 4 + (uint64_t)(n + 7) / 8) return ss_fail(ctx, SS_ERR_CAPACITY, "visibility output too small");
    SS_TRY(ss_scratch_reset(ctx));
    cudaStream_t s = ctx->stream;
    if (n) {
        SS_CUDA(ctx, ss_launch((k_abs_pack1<float>), dim3(grid_for(ctx, (n + 7) / 8)), dim3(256), 0, s, vis, n, out + 4));
        SS_CHECK_LAUNCH(ctx);
    }
    // '<I' count header and the length (a kernel: no host staging, no sync)
    SS_CUDA(ctx, ss_launch((k_vis_header), dim3(1), dim3(1), 0, s, n, out, out_len));
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}

}  // extern "C"
