// Client-side ingestion on the GPU: the decode half of
// the wire codec, bit-exact with the reference.
//
//   ss_decode_delta    ref protocol/delta.py:150-205 (decode_delta): LEB128
//                      gap varints decoded in parallel (terminator scan), the
//                      survivor indices by a prefix sum, codes dequantised in
//                      float64; malformed blocks set a status word instead of
//                      raising, checked in the reference's order
//   ss_apply_delta     ref protocol/delta.py:259-303 (advance_baseline +
//                      apply_delta): f32(f64(base) + dequant) on the touched
//                      rows, then the model attribute = baseline[:a];
//                      absolute attributes dequantised into (strided) columns
//   ss_decode_snapshot ref protocol/snapshot.py:85-168: every section of a
//                      profile-0 block (16-bit AABB means, 8/10/1-bit
//                      attributes, object-id varints) or a profile-1 copy
//
// The host side (protocol/ingest.py) parses headers, decompresses zlib
// blocks on the host exactly like the reference and checks every size it
// can know without reading the block; everything that needs the block's
// contents is checked here, on the device.
#include "ss_internal.cuh"

namespace {

enum { A_MEANS = 0, A_LS, A_QUAT, A_OPAC, A_DC, A_REST, A_VIS };

// ref quantize.py:20-24: lo + (code / levels) * (hi - lo), IEEE double ops
__device__ __forceinline__ double dequant(uint32_t code, double lo, double hi, int bits) {
    const double levels = (double)((1u << bits) - 1u);
    return da(lo, dm(dd((double)code, levels), ds(hi, lo)));
}

// code e of a packed stream: 16-bit little endian, bytes, or LSB-first bits
__device__ __forceinline__ uint32_t code_at(const uint8_t* p, int64_t e, int bits) {
    if (bits == 16) return (uint32_t)p[2 * e] | ((uint32_t)p[2 * e + 1] << 8);
    if (bits == 8) return p[e];
    const int64_t bit0 = e * bits;
    uint32_t v = 0;
    for (int b = 0; b < bits; ++b) {
        const int64_t bi = bit0 + b;
        v |= (uint32_t)((p[bi >> 3] >> (bi & 7)) & 1u) << b;
    }
    return v;
}

__device__ __forceinline__ int64_t col_off(const ss_delta_apply& a, int d) {
    return (int64_t)(d / a.inner) * a.outer + d % a.inner + a.col0;
}

// ---------------------------------------------------------------- varints
// Terminator bytes (high bit clear) end a varint; an exclusive scan of the
// terminator flags numbers the varints, so every varint is assembled
// independently.  Errors follow decode_varints (quantize.py:74-96): a varint
// of 11+ bytes is "too long" at its 10th byte; running out of bytes first is
// "truncated".
__global__ void k_term_flags(const uint8_t* __restrict__ b, int64_t n, uint8_t* __restrict__ term) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        term[i] = (b[i] & 0x80) == 0;
}

__global__ void k_term_pos(const uint8_t* __restrict__ term, const uint64_t* __restrict__ tidx, int64_t n,
                           int64_t count, int64_t* __restrict__ tpos) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (term[i] && (int64_t)tidx[i] < count) tpos[tidx[i]] = i;
}

// value v of the first min(count, T) varints; first_bad = lowest v with 11+
// bytes or a value beyond 64 bits
__global__ void k_varint_values(const uint8_t* __restrict__ b, const int64_t* __restrict__ tpos,
                                const uint64_t* __restrict__ total, int64_t count, uint64_t* __restrict__ vals,
                                unsigned long long* __restrict__ first_bad) {
    const int64_t m = min(count, (int64_t)*total);
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < m; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t start = v ? tpos[v - 1] + 1 : 0, end = tpos[v];
        if (end - start + 1 > 10) {
            atomicMin(first_bad, (unsigned long long)v);
            continue;
        }
        uint64_t val = 0;
        bool over = false;
        for (int64_t j = start; j <= end; ++j) {
            const uint64_t part = b[j] & 0x7Fu;
            const int sh = 7 * (int)(j - start);
            if (sh == 63 && part > 1) over = true;
            val |= part << sh;
        }
        if (over) atomicMin(first_bad, (unsigned long long)v);
        vals[v] = val;
    }
}

// one thread: the decode status of the varint run and its end offset
__global__ void k_varint_finish(const int64_t* __restrict__ tpos, const uint64_t* __restrict__ total, int64_t count,
                                int64_t n, const unsigned long long* __restrict__ first_bad,
                                ss_ingest_status* __restrict__ st) {
    if (st->code) return;
    const int64_t T = (int64_t)*total;
    if (*first_bad != ~0ull) {
        st->code = SS_INGEST_VARINT_TOO_LONG;
        return;
    }
    if (T < count) {
        const int64_t start = T ? tpos[T - 1] + 1 : 0;
        st->code = n - start >= 10 ? SS_INGEST_VARINT_TOO_LONG : SS_INGEST_VARINT_TRUNCATED;
        return;
    }
    st->offset = count ? tpos[count - 1] + 1 : 0;
}

// Decode `count` varints from b[0, n) into vals; status / end offset in st.
int decode_varints(ss_ctx* ctx, const uint8_t* b, int64_t n, int64_t count, uint64_t* vals, ss_ingest_status* st) {
    cudaStream_t s = ctx->stream;
    if (count == 0) return SS_OK;
    const int64_t na = n > 0 ? n : 1;
    uint8_t* term = SS_SCRATCH(ctx, uint8_t, na);
    uint64_t* tidx = SS_SCRATCH(ctx, uint64_t, na);
    uint64_t* total = SS_SCRATCH(ctx, uint64_t, 1);
    int64_t* tpos = SS_SCRATCH(ctx, int64_t, count);
    unsigned long long* bad = SS_SCRATCH(ctx, unsigned long long, 1);
    if (!term || !tidx || !total || !tpos || !bad) return SS_ERR_CUDA;
    SS_CUDA(ctx, cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
    SS_CUDA(ctx, cudaMemsetAsync(total, 0, sizeof(uint64_t), s));
    const int g = (int)min((n + 255) / 256, (int64_t)ctx->num_sms * 16) + 1;
    if (n > 0) {
        k_term_flags<<<g, 256, 0, s>>>(b, n, term);
        SS_CHECK_LAUNCH(ctx);
        SS_TRY(ss_scan_u8_to_u64(ctx, term, tidx, n, total));
        k_term_pos<<<g, 256, 0, s>>>(term, tidx, n, count, tpos);
        SS_CHECK_LAUNCH(ctx);
    }
    const int gv = (int)min((count + 255) / 256, (int64_t)ctx->num_sms * 16) + 1;
    k_varint_values<<<gv, 256, 0, s>>>(b, tpos, total, count, vals, bad);
    SS_CHECK_LAUNCH(ctx);
    k_varint_finish<<<1, 1, 0, s>>>(tpos, total, count, n, bad, st);
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}

// ---------------------------------------------------------------- delta decode
// survivor index i_v = sum_{u <= v} (gap_u + 1) - 1 (delta.py:180); a gap that
// does not fit 32 bits puts the index past any valid row count
__global__ void k_gap_plus1(const uint64_t* __restrict__ gaps, int64_t k, const ss_ingest_status* __restrict__ st,
                            uint32_t* __restrict__ g1) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < k; v += (int64_t)gridDim.x * blockDim.x)
        g1[v] = st->code ? 0u : (gaps[v] >= 0xfffffffeull ? 0xffffffffu : (uint32_t)(gaps[v] + 1));
}

__global__ void k_sparse_indices(const uint64_t* __restrict__ excl, const uint32_t* __restrict__ g1, int64_t k,
                                 int64_t count, int64_t block_len, int64_t code_bytes,
                                 int64_t* __restrict__ idx, ss_ingest_status* __restrict__ st) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < k; v += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t i = excl[v] + g1[v] - 1;
        idx[v] = (int64_t)i;
        if (v == k - 1 && st->code == 0) {
            if (i >= (uint64_t)count) st->code = SS_INGEST_INDEX_RANGE;               // delta.py:181-182
            else if (st->offset + code_bytes > block_len) st->code = SS_INGEST_CODES_TRUNCATED;  // delta.py:58-60
        }
    }
}

__global__ void k_delta_values(ss_delta_apply a, int64_t rows, const ss_ingest_status* __restrict__ st,
                               double* __restrict__ out) {
    if (st->code) return;
    const uint8_t* codes = a.block + (a.mode == 1 ? st->offset : 0);
    const int bits = a.bits;
    const int64_t n = rows * a.dims;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t c = code_at(codes, e, bits);
        out[e] = a.attribute_id == A_VIS ? (double)c : dequant(c, a.lo, a.hi, bits);
    }
}

// ---------------------------------------------------------------- delta apply
__global__ void k_apply_dense_residual(ss_delta_apply a, const ss_ingest_status* __restrict__ st) {
    if (st->code) return;
    const int64_t n = a.count * a.dims;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const double v = dequant(code_at(a.block, e, a.bits), a.lo, a.hi, a.bits);
        const float nb = __double2float_rn(da((double)a.baseline[e], v));  // delta.py:263
        a.baseline[e] = nb;
        const int64_t row = e / a.dims;
        a.target[row * a.row_stride + col_off(a, (int)(e - row * a.dims))] = nb;
    }
}

__global__ void k_apply_sparse_residual(ss_delta_apply a, const int64_t* __restrict__ idx,
                                        const ss_ingest_status* __restrict__ st) {
    if (st->code) return;
    const uint8_t* codes = a.block + st->offset;
    const int64_t n = a.k * a.dims;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = e / a.dims;
        const int d = (int)(e - s * a.dims);
        const double v = dequant(code_at(codes, e, a.bits), a.lo, a.hi, a.bits);
        float* p = a.baseline + idx[s] * a.dims + d;
        *p = __double2float_rn(da((double)*p, v));  // delta.py:265
    }
}

// model attribute[:a] = baseline[:a] (delta.py:285)
__global__ void k_copy_baseline(ss_delta_apply a, const ss_ingest_status* __restrict__ st) {
    if (st->code) return;
    const int64_t n = a.count * a.dims;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e / a.dims;
        a.target[row * a.row_stride + col_off(a, (int)(e - row * a.dims))] = a.baseline[e];
    }
}

__global__ void k_apply_absolute(ss_delta_apply a, const ss_ingest_status* __restrict__ st) {
    if (st->code) return;
    const int64_t n = a.count * a.dims;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t c = code_at(a.block, e, a.bits);
        const float v = a.attribute_id == A_VIS ? (float)c : __double2float_rn(dequant(c, a.lo, a.hi, a.bits));
        const int64_t row = e / a.dims;
        a.target[row * a.row_stride + col_off(a, (int)(e - row * a.dims))] = v;  // delta.py:287-301
    }
}

inline int grid_for(ss_ctx* ctx, int64_t n) {
    const int64_t g = (n + 255) / 256;
    const int64_t cap = (int64_t)ctx->num_sms * 16;
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

int check_apply_args(ss_ctx* ctx, const ss_delta_apply* a) {
    if (!a || !a->status) return ss_fail(ctx, SS_ERR_INVALID, "null argument");
    if (a->attribute_id < 0 || a->attribute_id > 6) return ss_fail(ctx, SS_ERR_PROTOCOL, "unknown attribute id");
    if (a->mode < 0 || a->mode > 2) return ss_fail(ctx, SS_ERR_PROTOCOL, "unknown delta mode");
    if (a->dims < 1 || a->count < 0 || a->k < 0 || a->k > a->count) return ss_fail(ctx, SS_ERR_INVALID, "bad shape");
    if (a->bits != 1 && a->bits != 8 && a->bits != 10 && a->bits != 16) return ss_fail(ctx, SS_ERR_INVALID, "bad bits");
    if (a->mode < 2 && a->attribute_id > A_LS) return ss_fail(ctx, SS_ERR_PROTOCOL, "not a residual attribute");
    if (a->inner < 1) return ss_fail(ctx, SS_ERR_INVALID, "bad column geometry");
    return SS_OK;
}

}  // namespace

extern "C" {

int ss_decode_delta(ss_ctx* ctx, const ss_delta_apply* a, int64_t* indices_out, double* values_out) {
    if (!ctx) return SS_ERR_INVALID;
    SS_TRY(check_apply_args(ctx, a));
    SS_TRY(ss_scratch_reset(ctx));
    cudaStream_t s = ctx->stream;
    SS_CUDA(ctx, cudaMemsetAsync(a->status, 0, sizeof(ss_ingest_status), s));
    if (a->mode == 1 && a->k > 0) {
        if (!indices_out) return ss_fail(ctx, SS_ERR_INVALID, "sparse decode needs indices_out");
        uint64_t* gaps = SS_SCRATCH(ctx, uint64_t, a->k);
        uint32_t* g1 = SS_SCRATCH(ctx, uint32_t, a->k);
        uint64_t* excl = SS_SCRATCH(ctx, uint64_t, a->k);
        uint64_t* tot = SS_SCRATCH(ctx, uint64_t, 1);
        if (!gaps || !g1 || !excl || !tot) return SS_ERR_CUDA;
        SS_TRY(decode_varints(ctx, a->block, a->block_len, a->k, gaps, a->status));
        k_gap_plus1<<<grid_for(ctx, a->k), 256, 0, s>>>(gaps, a->k, a->status, g1);
        SS_CHECK_LAUNCH(ctx);
        SS_TRY(ss_scan_u32_to_u64(ctx, g1, excl, a->k, tot));
        const int64_t cb = a->bits == 16 ? 2 : 1;
        k_sparse_indices<<<grid_for(ctx, a->k), 256, 0, s>>>(excl, g1, a->k, a->count, a->block_len,
                                                             a->k * a->dims * cb, indices_out, a->status);
        SS_CHECK_LAUNCH(ctx);
    }
    if (values_out) {
        const int64_t rows = a->mode == 1 ? a->k : a->count;
        if (rows > 0) {
            k_delta_values<<<grid_for(ctx, rows * a->dims), 256, 0, s>>>(*a, rows, a->status, values_out);
            SS_CHECK_LAUNCH(ctx);
        }
    }
    return SS_OK;
}

int ss_apply_delta(ss_ctx* ctx, const ss_delta_apply* a, const int64_t* indices) {
    if (!ctx) return SS_ERR_INVALID;
    SS_TRY(check_apply_args(ctx, a));
    if (a->count > 0 && !a->target) return ss_fail(ctx, SS_ERR_INVALID, "target is required");
    if (a->mode < 2 && a->count > 0 && !a->baseline) return ss_fail(ctx, SS_ERR_INVALID, "baseline is required");
    if (a->mode == 1 && a->k > 0 && !indices) return ss_fail(ctx, SS_ERR_INVALID, "indices are required");
    cudaStream_t s = ctx->stream;
    const int64_t n = a->count * a->dims;
    if (n == 0) return SS_OK;
    if (a->mode == 0) {
        k_apply_dense_residual<<<grid_for(ctx, n), 256, 0, s>>>(*a, a->status);
    } else if (a->mode == 1) {
        if (a->k > 0) {
            k_apply_sparse_residual<<<grid_for(ctx, a->k * a->dims), 256, 0, s>>>(*a, indices, a->status);
            SS_CHECK_LAUNCH(ctx);
        }
        k_copy_baseline<<<grid_for(ctx, n), 256, 0, s>>>(*a, a->status);
    } else {
        k_apply_absolute<<<grid_for(ctx, n), 256, 0, s>>>(*a, a->status);
    }
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- snapshot
namespace {

__global__ void k_snap_dequant(const uint8_t* __restrict__ codes, int64_t n_codes, int bits, int per_row,
                               int col_mod, double lo0, double hi0, double lo1, double hi1, double lo2, double hi2,
                               float* __restrict__ out, int64_t row_stride, int inner, int outer, int col0) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_codes; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e / per_row;
        const int d = (int)(e - row * per_row);
        double lo = lo0, hi = hi0;
        if (col_mod == 3) {  // per-axis AABB range of the means
            const int ax = d % 3;
            lo = ax == 0 ? lo0 : (ax == 1 ? lo1 : lo2);
            hi = ax == 0 ? hi0 : (ax == 1 ? hi1 : hi2);
        }
        const uint32_t c = code_at(codes, e, bits);
        const float v = bits == 1 ? (float)c : __double2float_rn(dequant(c, lo, hi, bits));
        out[row * row_stride + (int64_t)(d / inner) * outer + d % inner + col0] = v;
    }
}

__global__ void k_ids_from_varints(const uint64_t* __restrict__ v, int64_t n, const ss_ingest_status* __restrict__ st,
                                   int32_t* __restrict__ ids) {
    if (st->code) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        ids[i] = (int32_t)(uint32_t)v[i];  // astype(np.int32) keeps the low 32 bits (snapshot.py:154)
}

}  // namespace

extern "C" int ss_decode_snapshot(ss_ctx* ctx, const ss_snapshot_decode* d) {
    if (!ctx || !d || !d->status) return SS_ERR_INVALID;
    const ss_model& m = d->model;
    const int64_t n = m.count;
    if (n < 0 || m.sh_degree < 0 || m.sh_degree > 3) return ss_fail(ctx, SS_ERR_INVALID, "bad snapshot shape");
    SS_TRY(ss_scratch_reset(ctx));
    cudaStream_t s = ctx->stream;
    SS_CUDA(ctx, cudaMemsetAsync(d->status, 0, sizeof(ss_ingest_status), s));
    if (n == 0) return SS_OK;
    const int B = (m.sh_degree + 1) * (m.sh_degree + 1);
    const uint8_t* p = d->block;
    if (d->profile_id == 1) {  // lossless: float32 / int32 sections copied in place (snapshot.py:119-126)
        const size_t sz[7] = {12, 12, 16, 4, (size_t)12 * B, 4, 4};
        void* dst[7] = {m.means, m.log_scales, m.quaternions, m.logit_opacities, m.sh_coeffs, m.light_visibility,
                        m.object_ids};
        for (int i = 0; i < 7; ++i) {
            SS_CUDA(ctx, cudaMemcpyAsync(dst[i], p, sz[i] * n, cudaMemcpyDeviceToDevice, s));
            p += sz[i] * n;
        }
        return SS_OK;
    }
    // profile 0 (snapshot.py:127-154): sections in wire order
    const int g = (int)min((3 * B * n + 255) / 256, (int64_t)ctx->num_sms * 16);
    auto launch = [&](const uint8_t* codes, int64_t n_codes, int bits, int per_row, int col_mod, double lo,
                      double hi, float* out, int64_t row_stride, int inner, int outer, int col0) {
        k_snap_dequant<<<g, 256, 0, s>>>(codes, n_codes, bits, per_row, col_mod, col_mod == 3 ? d->aabb_lo[0] : lo,
                                         col_mod == 3 ? d->aabb_hi[0] : hi, d->aabb_lo[1], d->aabb_hi[1],
                                         d->aabb_lo[2], d->aabb_hi[2], out, row_stride, inner, outer, col0);
    };
    launch(p, 3 * n, 16, 3, 3, 0, 0, m.means, 3, 3, 0, 0);
    p += 6 * n;
    SS_CHECK_LAUNCH(ctx);
    launch(p, 3 * n, 8, 3, 0, -10.0, 2.0, m.log_scales, 3, 3, 0, 0);
    p += 3 * n;
    SS_CHECK_LAUNCH(ctx);
    launch(p, 4 * n, 10, 4, 0, -1.0, 1.0, m.quaternions, 4, 4, 0, 0);
    p += (4 * n * 10 + 7) / 8;
    SS_CHECK_LAUNCH(ctx);
    launch(p, n, 8, 1, 0, -8.0, 8.0, m.logit_opacities, 1, 1, 0, 0);
    p += n;
    SS_CHECK_LAUNCH(ctx);
    launch(p, 3 * n, 8, 3, 0, -4.0, 4.0, m.sh_coeffs, 3 * B, 1, B, 0);  // sh[:, :, 0]
    p += 3 * n;
    SS_CHECK_LAUNCH(ctx);
    if (B > 1) {
        launch(p, 3 * (B - 1) * n, 8, 3 * (B - 1), 0, -1.0, 1.0, m.sh_coeffs, 3 * B, B - 1, B, 1);  // sh[:, :, 1:]
        p += 3 * (int64_t)(B - 1) * n;
        SS_CHECK_LAUNCH(ctx);
    }
    launch(p, n, 1, 1, 0, 0.0, 1.0, m.light_visibility, 1, 1, 0, 0);
    p += (n + 7) / 8;
    SS_CHECK_LAUNCH(ctx);
    // object ids: n varints after the fixed sections (snapshot.py:153)
    const int64_t off = p - d->block;
    uint64_t* vals = SS_SCRATCH(ctx, uint64_t, n);
    if (!vals) return SS_ERR_CUDA;
    SS_TRY(decode_varints(ctx, p, d->block_len - off, n, vals, d->status));
    k_ids_from_varints<<<grid_for(ctx, n), 256, 0, s>>>(vals, n, d->status, m.object_ids);
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}
