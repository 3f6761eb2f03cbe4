// Batched delta encoder: one server tick's attribute deltas (ref
// pkg/src/splatstream/server.py:488-493 -> protocol/delta.py:72-137) in ONE
// launch of k_tick_fused, whatever the number of attributes.  Blocks, in
// dispatch order:
//
//   residual scans  every residual (job, 2048-row chunk): chunk stats (kept
//                   rows, max|r| over all / kept rows, first / last kept row,
//                   varint bytes of the chunk's internal gaps); the last chunk
//                   of a job to finish plans it (mode k < rows/2, f32 range m,
//                   per-chunk prefixes, header, payload length) and releases
//                   the job's flag
//   absolute jobs   every absolute (job, chunk): quantize + pack straight
//                   into the payload (covers the plan tail)
//   residual emits  wait for their job's flag, then dense quantize, or sparse
//                   varint gaps + codes; advanced baseline f32(f64(base) + deq)
//
// (TK_ORDER 1 runs the residual emits before the absolute jobs instead, so
// an emit re-reads its chunk's cur / base while they are still in L2.)
// A block's role is its ticket from an atomic counter taken when it starts
// (not blockIdx.x, whose dispatch order CUDA does not guarantee): every scan
// block an emit block waits for holds a smaller ticket, so it has already
// started and will finish -- the forward-progress argument of the radix
// sort's decoupled look-back (ss_sort.cu takes its tiles the same way).
//
// Inputs may be strided views of the model (SH DC / SH rest are read in place
// from the (N, 3, B) coefficient array).  Arithmetic is the bit-exact float64
// of ss_codec.cu; the output bytes equal the reference's with
// compression_id 0.  No host synchronisation.
#include "ss_internal.cuh"

namespace {

constexpr int TK_THREADS = 256;
constexpr int TK_ITEMS = 8;
constexpr int TK_CHUNK = TK_THREADS * TK_ITEMS;  // rows per block
constexpr int TK_MAX_JOBS = 8;
#ifndef EMIT_U
#define EMIT_U 3
#endif
// EMIT_U: float4 steps in flight per thread: 3 x 2 rounds = a full dims-3 chunk

struct QParams {
    double lo, hi, span, inv_span, levels, inv_levels, dspan;  // dspan = hi - lo (dequantizer)
    double p2scale;  // levels / span when hi > lo and span is a power of two (exact), else 0
    int bits;
};

__host__ __device__ inline QParams make_q(double lo, double hi, int bits) {
    QParams p;
    p.lo = lo;
    p.hi = hi;
    p.bits = bits;
    p.levels = (double)((1u << bits) - 1u);
    p.inv_levels = 1.0 / p.levels;
    p.span = hi > lo ? hi - lo : 1.0;
    p.inv_span = 1.0 / p.span;
    p.dspan = hi - lo;
    int ex = 0;
    p.p2scale = (hi > lo && frexp(p.span, &ex) == 0.5) ? p.levels * p.inv_span : 0.0;
    return p;
}

struct Job {
    const void* cur;       // element (row, d) at cur + row*row_stride + (d / inner) * outer + d % inner + col0
    const void* base;      // residual only; same geometry as cur
    float* new_base;       // residual only, dense (rows, dims) float32; may alias base
    uint8_t* out;
    uint64_t* out_len;
    int64_t rows;
    int64_t row_stride;
    int dims, inner, outer, col0;
    int attr, bits, residual, f64;
    double gate, qlo, qhi;
    float gate_lo, gate_hi;  // float32 bracket of gate: rmax32 > hi keeps, < lo drops, else exact fp64 test
    QParams q;             // absolute quantizer
    int64_t chunk0;        // first global chunk of this job
    int64_t nchunks;
    // residual scratch
    unsigned long long* g;  // [0] count, [1] max_all, [2] max_keep (f32 bits of max|r|), [3] finished chunks
    uint32_t* ck;           // per chunk: kept rows
    int64_t* cfirst;        // per chunk: first kept row (-1)
    int64_t* clast;         // per chunk: last kept row (-1)
    uint32_t* cvar;         // per chunk: varint bytes of gaps after the chunk's first survivor
    uint32_t* cmax;         // per chunk: [2c] f32 bits of max|r| over all rows, [2c+1] over kept rows
    uint32_t* cnt_pre;      // per chunk: survivors before the chunk
    uint64_t* var_pre;      // per chunk: varint bytes before the chunk
    int64_t* prev_last;     // per chunk: last kept row before the chunk (-1)
    double* m;              // chosen range
    QParams* rq;            // residual quantizer over [-m, m] (set by k_tick_plan)
    int* mode;              // 0 dense, 1 sparse
};

struct Batch {
    Job j[TK_MAX_JOBS];
    int n;
};

__device__ __forceinline__ double q_dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double q_da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double q_ds(double a, double b) { return __dsub_rn(a, b); }

// Correctly rounded a / b from y = RN(1/b): q = RN(a y), r = a - b q (exact
// by FMA), RN(q + r y) = RN(a / b)  (Markstein's theorem; our quotients are
// normal numbers in [0, 65535]).  Replaces the generic __ddiv_rn sequence
// (reciprocal + Newton + special-case path) in the per-element hot loop.
__device__ __forceinline__ double div_rn(double a, double b, double y) {
    const double q = __dmul_rn(a, y);
    const double r = __fma_rn(-b, q, a);
    return __fma_rn(r, y, q);
}

// numpy's maximum/minimum for non-NaN inputs (a >= b ? a : b), as plain
// compare + select: fmax/fmin compile to ~6 instructions each for doubles
__device__ __forceinline__ double np_max(double a, double b) { return a >= b ? a : b; }
__device__ __forceinline__ double np_min(double a, double b) { return a <= b ? a : b; }

// ref quantize.py:8-17, bit-exact.  For hi >= lo, clip(v) - lo <= RN(hi - lo)
// by monotone rounding, so t already lies in [0, 1] and its clip is a no-op.
__device__ __forceinline__ uint32_t quant(double v, const QParams& p) {
    const double c = np_min(np_max(v, p.lo), p.hi);
    // power-of-two span: x / span is exact, so RN(RN(x / span) * levels) ==
    // RN(x * (levels / span)) -- one multiply, and rint + convert in one step
    if (p.p2scale != 0.0) return (uint32_t)__double2int_rn(q_dm(q_ds(c, p.lo), p.p2scale));
    double t = div_rn(q_ds(c, p.lo), p.span, p.inv_span);
    if (!(p.hi >= p.lo)) t = np_min(np_max(t, 0.0), 1.0);
    return (uint32_t)rint(q_dm(t, p.levels));
}

// ref quantize.py:20-24, bit-exact
__device__ __forceinline__ double dequant(uint32_t code, const QParams& p) {
    return q_da(p.lo, q_dm(div_rn((double)code, p.levels, p.inv_levels), p.dspan));
}

// dequantised value of an integer-valued code held as a double
__device__ __forceinline__ double dequant_d(double cd, const QParams& p) {
    return q_da(p.lo, q_dm(div_rn(cd, p.levels, p.inv_levels), p.dspan));
}

// Residual quantizer over [-m, m] (ref quantize.py:8-24 via delta.py:109-110,
// 117-118), bit-exact with the clip moved after the rounding: RN is monotone,
// so r > m gives t >= 1 and a code >= levels, r < -m gives t <= 0 and a code
// <= 0, and clamping the integer code reproduces clip-then-quantize; m == 0
// (span 1, every residual below the smallest subnormal) codes 0.
__device__ __forceinline__ int rquant(double r, const QParams& p) {
    const double t = div_rn(q_ds(r, p.lo), p.span, p.inv_span);
    const int code = __double2int_rn(q_dm(t, p.levels));
    return min(max(code, 0), (int)p.levels);
}
// advanced baseline f32(f64(base) + dequant(code))
__device__ __forceinline__ float radvance(double b, int code, const QParams& p) {
    return __double2float_rn(q_da(b, dequant_d((double)code, p)));
}

__device__ __forceinline__ int vlen(uint64_t v) {
    int n = 1;
    while (v >= 0x80) {
        v >>= 7;
        ++n;
    }
    return n;
}

__device__ __forceinline__ void vput(uint8_t* p, uint64_t v) {
    while (v >= 0x80) {
        *p++ = (uint8_t)(v & 0x7F) | 0x80;
        v >>= 7;
    }
    *p = (uint8_t)v;
}

__device__ __forceinline__ void put32(uint8_t* p, uint32_t v) {
    p[0] = v & 0xff;
    p[1] = (v >> 8) & 0xff;
    p[2] = (v >> 16) & 0xff;
    p[3] = v >> 24;
}

// column offsets of a job's dims within a row, built once per block
constexpr int TK_MAX_DIMS = 64;
__device__ __forceinline__ void build_cols(const Job& J, int* s_col) {
    for (int d = threadIdx.x; d < J.dims; d += blockDim.x) s_col[d] = (d / J.inner) * J.outer + d % J.inner + J.col0;
    __syncthreads();
}

#define LDX(p, row, d) (J.f64 ? ((const double*)(p))[(row) * J.row_stride + s_col[d]] \
                              : (double)((const float*)(p))[(row) * J.row_stride + s_col[d]])

__device__ __forceinline__ int find_job(const Batch& B, int64_t chunk) {
    int k = 0;
    for (int i = 0; i < B.n; ++i)
        if (chunk >= B.j[i].chunk0 && chunk < B.j[i].chunk0 + B.j[i].nchunks) k = i;
    return k;
}

// ---------------------------------------------------------------- scan
template <typename T>
__device__ __forceinline__ void scan_absolute(const Job& J, const int* s_col, int64_t r0, int64_t r1) {
    uint8_t* blk = J.out + 12;
    const T* cur = (const T*)J.cur;
    const bool contig = J.row_stride == J.dims && J.inner == J.dims && J.col0 == 0;
    if (J.attr == 6) {  // 1-bit visibility (dims 1): 8 rows per byte, chunks are byte aligned
        for (int64_t byte = r0 / 8 + threadIdx.x; byte * 8 < r1; byte += TK_THREADS) {
            uint8_t v = 0;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int64_t row = byte * 8 + t;
                if (row < r1 && (double)__ldcs(&cur[row * J.row_stride + s_col[0]]) >= 0.5) v |= (uint8_t)(1u << t);
            }
            blk[byte] = v;
        }
    } else if (J.bits == 10) {  // 4 codes -> 5 bytes per row (dims == 4)
        for (int64_t row = r0 + threadIdx.x; row < r1; row += TK_THREADS) {
            uint64_t w = 0;
#pragma unroll
            for (int d = 0; d < 4; ++d) w |= (uint64_t)quant((double)__ldcs(&cur[row * J.row_stride + s_col[d]]), J.q) << (10 * d);
#pragma unroll
            for (int b = 0; b < 5; ++b) blk[row * 5 + b] = (uint8_t)(w >> (8 * b));
        }
    } else if (contig) {  // 8-bit codes, elementwise, 4 loads in flight
        const int64_t e1 = r1 * J.dims;
        for (int64_t e = r0 * J.dims + threadIdx.x; e < e1; e += 4 * TK_THREADS) {
            T v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (e + u * TK_THREADS < e1) v[u] = __ldcs(&cur[e + u * TK_THREADS]);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (e + u * TK_THREADS < e1) blk[e + u * TK_THREADS] = (uint8_t)quant((double)v[u], J.q);
        }
    } else if (J.dims == 3) {  // 8-bit codes of a strided 3-wide view (SH DC): prefetch 4 rows
        const int c0 = s_col[0], c1 = s_col[1], c2 = s_col[2];
        for (int64_t row = r0 + threadIdx.x; row < r1; row += 4 * TK_THREADS) {
            T v[4][3];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t rr = row + u * TK_THREADS;
                if (rr < r1) {
                    const T* src = cur + rr * J.row_stride;
                    v[u][0] = __ldcs(&src[c0]);
                    v[u][1] = __ldcs(&src[c1]);
                    v[u][2] = __ldcs(&src[c2]);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t rr = row + u * TK_THREADS;
                if (rr < r1)
#pragma unroll
                    for (int d = 0; d < 3; ++d) blk[rr * 3 + d] = (uint8_t)quant((double)v[u][d], J.q);
            }
        }
    } else {  // 8-bit codes of a strided view, one row per thread
        for (int64_t row = r0 + threadIdx.x; row < r1; row += TK_THREADS) {
            const T* src = cur + row * J.row_stride;
            uint8_t* dst = blk + row * J.dims;
            for (int d = 0; d < J.dims; ++d) dst[d] = (uint8_t)quant((double)src[s_col[d]], J.q);
        }
    }
}

// exact fp64 gate test of one row (ref delta.py:95-96)
template <typename T>
__device__ __forceinline__ bool keep_exact(const T* cur, const T* base, int64_t row, int dims, double gate) {
    double rmax = 0.0;
    for (int d = 0; d < dims; ++d)
        rmax = np_max(rmax, fabs(q_ds((double)cur[row * dims + d], (double)base[row * dims + d])));
    return rmax >= gate;
}

// Per-row statistics: rm = RN32(max_d |r_d|) and keep = (max_d |r_d| >= gate)
// with r = f64(cur) - f64(base).  For float32 inputs the residual is formed in
// float32: RN32(a - b) = RN32(RN64(a - b)) for float32 a, b (the difference is
// exact in fp64 unless |b| < 2^-29 |a|, and then no float32 rounding boundary
// lies within an fp64 ulp of it), |.| and max commute with monotone
// rounding, so rm is exactly RN32 of the fp64 maximum; the gate is decided in
// float32 outside a 2^-20 relative band around it and in fp64 inside.
__device__ __forceinline__ float f_max(float a, float b) { return a >= b ? a : b; }

__device__ __forceinline__ bool gate_keep(float rm, const Job& J, const float* cur, const float* base, int64_t row) {
    if (rm > J.gate_hi) return true;
    if (rm < J.gate_lo) return false;
    return keep_exact<float>(cur, base, row, J.dims, J.gate);
}

template <typename T>
__device__ __forceinline__ void scan_residual(const Job& J, int64_t c, int64_t r0, int64_t r1) {
    __shared__ uint32_t s_keep[TK_CHUNK / 32];  // kept-row bitmap of this chunk
    __shared__ unsigned long long s_mall[TK_THREADS / 32], s_mkeep[TK_THREADS / 32];
    __shared__ uint32_t s_var[TK_THREADS / 32];
    const T* cur = (const T*)J.cur;
    const T* base = (const T*)J.base;
    const int dims = J.dims;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t mall = 0, mkeep = 0;  // f32 bits of non-negative maxima (ordered as integers)
    if (sizeof(T) == 4 && dims == 3 && r1 - r0 == TK_CHUNK) {
        // full chunk, dims 3: issue all 48 loads of the thread's 8 rows first
        const float* cf = (const float*)cur;
        const float* bf = (const float*)base;
        float cv[TK_ITEMS][3], bv[TK_ITEMS][3];
#pragma unroll
        for (int it = 0; it < TK_ITEMS; ++it) {
            const int64_t row = r0 + it * TK_THREADS + threadIdx.x;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                cv[it][d] = cf[row * 3 + d];
                bv[it][d] = bf[row * 3 + d];
            }
        }
#pragma unroll
        for (int it = 0; it < TK_ITEMS; ++it) {
            const int64_t row = r0 + it * TK_THREADS + threadIdx.x;
            float rm = 0.f;
#pragma unroll
            for (int d = 0; d < 3; ++d) rm = f_max(rm, fabsf(cv[it][d] - bv[it][d]));
            const bool keep = gate_keep(rm, J, cf, bf, row);
            const uint32_t bits = __float_as_uint(rm);
            mall = bits > mall ? bits : mall;
            if (keep) mkeep = bits > mkeep ? bits : mkeep;
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) s_keep[it * (TK_THREADS / 32) + warp] = bal;
        }
    } else
    for (int it = 0; it < TK_ITEMS; ++it) {
        const int64_t row = r0 + it * TK_THREADS + threadIdx.x;  // striped: coalesced per item
        bool keep = false;
        if (row < r1) {
            float rm;
            if constexpr (sizeof(T) == 4) {
                rm = 0.f;
                for (int d = 0; d < dims; ++d) rm = f_max(rm, fabsf(cur[row * dims + d] - base[row * dims + d]));
                keep = gate_keep(rm, J, (const float*)cur, (const float*)base, row);
            } else {
                double rmax = 0.0;
                for (int d = 0; d < dims; ++d) {
                    const int64_t e = row * dims + d;
                    rmax = np_max(rmax, fabs(q_ds((double)cur[e], (double)base[e])));
                }
                keep = rmax >= J.gate;
                rm = __double2float_rn(rmax);
            }
            const uint32_t bits = __float_as_uint(rm);
            mall = bits > mall ? bits : mall;
            if (keep) mkeep = bits > mkeep ? bits : mkeep;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_keep[it * (TK_THREADS / 32) + warp] = bal;
    }
    mall = __reduce_max_sync(0xffffffffu, mall);
    mkeep = __reduce_max_sync(0xffffffffu, mkeep);
    if (lane == 0) {
        s_mall[warp] = mall;
        s_mkeep[warp] = mkeep;
    }
    __syncthreads();
    // varint bytes of the gaps inside the chunk (first survivor excluded):
    // gaps inside a 32-row word are < 32 (one byte each), so a word costs
    // popc(bits) bytes plus the extra bytes of its first survivor's gap to
    // the nearest survivor in an earlier word
    uint32_t var = 0;
    if (threadIdx.x < TK_CHUNK / 32) {
        const int w = threadIdx.x;
        const uint32_t bits = s_keep[w];
        if (bits) {
            int64_t prev = -1;
            for (int k2 = w - 1; k2 >= 0; --k2)
                if (s_keep[k2]) {
                    prev = r0 + 32 * k2 + (31 - __clz(s_keep[k2]));
                    break;
                }
            const int64_t first = r0 + 32 * w + (__ffs(bits) - 1);
            var = __popc(bits) - 1 + (prev >= 0 ? vlen((uint64_t)(first - prev - 1)) : 0);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
    if (lane == 0) s_var[warp] = var;
    __syncthreads();
    if (warp == 0) {  // chunk summary from the 64 bitmap words, warp-parallel
        const uint32_t w0 = s_keep[lane], w1 = s_keep[32 + lane];
        const uint32_t cnt = __reduce_add_sync(0xffffffffu, __popc(w0) + __popc(w1));
        const unsigned nz0 = __ballot_sync(0xffffffffu, w0 != 0), nz1 = __ballot_sync(0xffffffffu, w1 != 0);
        int64_t first = -1, last = -1;
        if (nz0 | nz1) {
            const int fw = nz0 ? __ffs(nz0) - 1 : 32 + __ffs(nz1) - 1;
            const int lw = nz1 ? 32 + 31 - __clz(nz1) : 31 - __clz(nz0);
            first = r0 + 32 * fw + (__ffs(s_keep[fw]) - 1);
            last = r0 + 32 * lw + (31 - __clz(s_keep[lw]));
        }
        uint32_t vs = lane < TK_THREADS / 32 ? s_var[lane] : 0;
        vs = __reduce_add_sync(0xffffffffu, vs);
        const uint32_t ma = __reduce_max_sync(0xffffffffu, lane < TK_THREADS / 32 ? (uint32_t)s_mall[lane] : 0u);
        const uint32_t mk = __reduce_max_sync(0xffffffffu, lane < TK_THREADS / 32 ? (uint32_t)s_mkeep[lane] : 0u);
        if (lane == 0) {
            J.ck[c] = cnt;
            J.cfirst[c] = first;
            J.clast[c] = last;
            J.cvar[c] = vs;
            J.cmax[2 * c] = ma;  // reduced by the job's plan (no contended global atomics)
            J.cmax[2 * c + 1] = mk;
        }
    }
}

// ---------------------------------------------------------------- plan
// Run by the last block to finish a residual job's scan (or by k_tick_plan
// for a job without rows): mode decision (k < rows/2, delta.py:101), f32
// range m, per-chunk prefixes for the sparse writer, header, payload length.
// Chunk statistics written by other blocks are read with ld.global.cg (L2).

// inclusive block scan (sum) over TK_THREADS threads; returns the block total in *tot
__device__ __forceinline__ uint64_t plan_scan_sum(uint64_t v, uint64_t* tot) {
    __shared__ uint64_t ws[TK_THREADS / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    if (lane == 31) ws[w] = v;
    __syncthreads();
    uint64_t pre = 0, all = 0;
#pragma unroll
    for (int k = 0; k < TK_THREADS / 32; ++k) {
        const uint64_t x = ws[k];
        if (k < w) pre += x;
        all += x;
    }
    *tot = all;
    __syncthreads();
    return v + pre;
}

// inclusive block scan (max) of signed values
__device__ __forceinline__ long long plan_scan_max(long long v, long long* tot, long long* excl) {
    __shared__ long long ws[TK_THREADS / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o && t > v) v = t;
    }
    if (lane == 31) ws[w] = v;
    __syncthreads();
    long long pre = -1, all = -1;
#pragma unroll
    for (int k = 0; k < TK_THREADS / 32; ++k) {
        const long long x = ws[k];
        if (k < w && x > pre) pre = x;
        if (x > all) all = x;
    }
    long long up = __shfl_up_sync(0xffffffffu, v, 1);
    if (lane == 0) up = -1;
    *excl = up > pre ? up : pre;  // exclusive max (earlier threads of the block)
    *tot = all;
    __syncthreads();
    return v > pre ? v : pre;
}

__device__ void plan_job(const Job& J) {
    // survivors and maxima over the job's chunks (float bits order as integers)
    __shared__ unsigned long long s_k;
    __shared__ uint32_t s_ma, s_mk;
    {
        uint64_t kk = 0;
        uint32_t ma = 0, mk = 0;
        for (int64_t c = threadIdx.x; c < J.nchunks; c += TK_THREADS) {
            kk += __ldcg(&J.ck[c]);
            ma = max(ma, __ldcg(&J.cmax[2 * c]));
            mk = max(mk, __ldcg(&J.cmax[2 * c + 1]));
        }
        uint64_t tot;
        plan_scan_sum(kk, &tot);
        ma = __reduce_max_sync(0xffffffffu, ma);
        mk = __reduce_max_sync(0xffffffffu, mk);
        if (threadIdx.x == 0) s_ma = 0, s_mk = 0, s_k = tot;
        __syncthreads();
        if ((threadIdx.x & 31) == 0) {
            atomicMax(&s_ma, ma);
            atomicMax(&s_mk, mk);
        }
        __syncthreads();
    }
    const unsigned long long k = s_k;
    const int sparse = 2 * (int64_t)k < J.rows;  // k < rows * 0.5 (delta.py:101)
    double m;
    if (sparse) m = k ? (double)__uint_as_float(s_mk) : 0.0;
    else m = J.rows ? (double)__uint_as_float(s_ma) : 0.0;
    if (threadIdx.x == 0) {
        *J.mode = sparse;
        *J.m = m;
        QParams rq;
        rq.lo = -m;
        rq.hi = m;
        rq.bits = J.bits;
        rq.levels = (double)((1u << J.bits) - 1u);
        rq.inv_levels = 1.0 / rq.levels;
        rq.span = m > -m ? q_ds(m, -m) : 1.0;
        rq.inv_span = 1.0 / rq.span;
        rq.dspan = q_ds(m, -m);
        rq.p2scale = 0.0;  // residual codes use rquant
        *J.rq = rq;
    }
    uint64_t V = 0;
    if (sparse) {
        // per-chunk prefixes: survivors, varint bytes and the last kept row
        // before each chunk (block scans carried over rounds of TK_THREADS chunks)
        uint64_t kc = 0, vc = 0;
        long long lc = -1;
        for (int64_t c0 = 0; c0 < J.nchunks; c0 += TK_THREADS) {
            const int64_t c = c0 + threadIdx.x;
            const bool in = c < J.nchunks;
            const uint32_t ck = in ? __ldcg(&J.ck[c]) : 0;
            const long long cl = in && ck ? (long long)__ldcg(&J.clast[c]) : -1;
            uint64_t ktot;
            const uint64_t kin = plan_scan_sum(ck, &ktot);
            long long ltot, prev;
            plan_scan_max(cl, &ltot, &prev);
            if (prev < lc) prev = lc;
            const uint64_t vbytes = in && ck ? (uint64_t)vlen((uint64_t)(__ldcg(&J.cfirst[c]) - prev - 1)) + __ldcg(&J.cvar[c]) : 0;
            uint64_t vtot;
            const uint64_t vin = plan_scan_sum(vbytes, &vtot);
            if (in) {
                J.cnt_pre[c] = (uint32_t)(kc + kin - ck);
                J.var_pre[c] = vc + vin - vbytes;
                J.prev_last[c] = prev;
            }
            kc += ktot;
            vc += vtot;
            if (ltot > lc) lc = ltot;
        }
        V = vc;
    }
    if (threadIdx.x == 0) {
        const int cb = J.bits / 8;
        const uint64_t blen = sparse ? V + k * J.dims * cb : (uint64_t)J.rows * J.dims * cb;
        uint8_t* o = J.out;
        o[0] = (uint8_t)J.attr;
        o[1] = (uint8_t)sparse;
        o[2] = 0;
        o[3] = (uint8_t)J.dims;
        put32(o + 4, (uint32_t)J.rows);
        const float mf = (float)m;
        put32(o + 8, __float_as_uint(-mf));
        put32(o + 12, __float_as_uint(mf));
        int h = 16;
        if (sparse) {
            put32(o + 16, (uint32_t)k);
            h = 20;
        }
        put32(o + h, (uint32_t)blen);
        *J.out_len = h + 4 + blen;
        J.var_pre[J.nchunks] = V;  // total varint bytes (sparse code offset)
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // planned: release the job to its emit blocks
        __threadfence();
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&J.g[2]), "l"(1ull) : "memory");
    }
}

// an emit block of the fused launch waits for its job's plan
__device__ __forceinline__ void wait_planned(const Job& J) {
    unsigned long long f;
    if (threadIdx.x == 0) {
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(&J.g[2]) : "memory");
            if (f) break;
            __nanosleep(256);
        }
    }
    __syncthreads();
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(&J.g[2]) : "memory");
}

// an absolute job without rows: header only (mode 2, zero-length block)
__global__ void k_empty_header(Batch B, int job) {
    SS_PDL_WAIT();
    const Job& J = B.j[job];
    uint8_t* o = J.out;
    o[0] = (uint8_t)J.attr;
    o[1] = 2;
    o[2] = 0;
    o[3] = (uint8_t)J.dims;
    for (int k = 4; k < 12; ++k) o[k] = 0;
    *J.out_len = 12;
}

// a residual job without rows (no scan block runs its plan)
__global__ void __launch_bounds__(TK_THREADS) k_tick_plan(Batch B, int job) {
    SS_PDL_WAIT(); plan_job(B.j[job]); }

// ---------------------------------------------------------------- emit
template <typename T>
__device__ __forceinline__ void emit_dense(const Job& J, const QParams& rq, int64_t r0, int64_t r1) {
    // elementwise: residual code of element e and its advanced baseline
    const T* cur = (const T*)J.cur;
    const T* base = (const T*)J.base;
    const int64_t e1 = r1 * J.dims;
    if (sizeof(T) == 4 && J.bits == 8 && J.new_base &&
        (((uintptr_t)cur | (uintptr_t)base | (uintptr_t)J.new_base) & 15) == 0 && ((r0 * J.dims) & 3) == 0) {
        const int64_t v0 = r0 * J.dims / 4, v1 = e1 / 4;
        const float4* c4 = (const float4*)cur;
        const float4* b4 = (const float4*)base;
        float4* n4 = (float4*)J.new_base;
        uint8_t* blk = J.out + 20;
        for (int64_t v = v0 + threadIdx.x; v < v1; v += EMIT_U * TK_THREADS) {
            float4 cc[EMIT_U], bb[EMIT_U];
#pragma unroll
            for (int u = 0; u < EMIT_U; ++u) {
                const int64_t w = v + u * TK_THREADS;
                if (w < v1) {  // last use of cur/base: evict-first
                    cc[u] = __ldcs(&c4[w]);
                    bb[u] = __ldcs(&b4[w]);
                }
            }
#pragma unroll
            for (int u = 0; u < EMIT_U; ++u) {
                const int64_t w = v + u * TK_THREADS;
                if (w >= v1) continue;
                const float cs[4] = {cc[u].x, cc[u].y, cc[u].z, cc[u].w};
                const float bs[4] = {bb[u].x, bb[u].y, bb[u].z, bb[u].w};
                uint32_t packed = 0;
                float nb[4];
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const int code = rquant(q_ds((double)cs[kk], (double)bs[kk]), rq);
                    packed |= (uint32_t)code << (8 * kk);
                    nb[kk] = radvance((double)bs[kk], code, rq);
                }
                __stcs(&n4[w], make_float4(nb[0], nb[1], nb[2], nb[3]));
                *reinterpret_cast<uint32_t*>(blk + 4 * w) = packed;  // 20 + 4w: 4-byte aligned
            }
        }
        for (int64_t e = 4 * v1 + threadIdx.x; e < e1; e += TK_THREADS) {
            const double b = (double)base[e];
            const int code = rquant(q_ds((double)cur[e], b), rq);
            blk[e] = (uint8_t)code;
            J.new_base[e] = radvance(b, code, rq);
        }
        return;
    }
    if (sizeof(T) == 4 && J.bits == 16 && J.new_base &&
        (((uintptr_t)cur | (uintptr_t)base | (uintptr_t)J.new_base) & 15) == 0 && ((r0 * J.dims) & 3) == 0) {
        // 4 elements per thread-step: float4 loads/stores, 8-byte code stores; 4 steps in flight
        const int64_t v0 = r0 * J.dims / 4, v1 = e1 / 4;
        const float4* c4 = (const float4*)cur;
        const float4* b4 = (const float4*)base;
        float4* n4 = (float4*)J.new_base;
        uint2* code4 = (uint2*)(J.out + 24);  // 8-byte aligned view starting 4 bytes past the block
        uint16_t* blk = (uint16_t*)(J.out + 20);
        for (int64_t v = v0 + threadIdx.x; v < v1; v += EMIT_U * TK_THREADS) {
            float4 cc[EMIT_U], bb[EMIT_U];
#pragma unroll
            for (int u = 0; u < EMIT_U; ++u) {
                const int64_t w = v + u * TK_THREADS;
                if (w < v1) {  // last use of cur/base: evict-first
                    cc[u] = __ldcs(&c4[w]);
                    bb[u] = __ldcs(&b4[w]);
                }
            }
#pragma unroll
            for (int u = 0; u < EMIT_U; ++u) {
                const int64_t w = v + u * TK_THREADS;
                if (w >= v1) continue;
                const float cs[4] = {cc[u].x, cc[u].y, cc[u].z, cc[u].w};
                const float bs[4] = {bb[u].x, bb[u].y, bb[u].z, bb[u].w};
                uint32_t code[4];
                float nb[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int cq = rquant(q_ds((double)cs[k], (double)bs[k]), rq);
                    code[k] = (uint32_t)cq;
                    nb[k] = radvance((double)bs[k], cq, rq);
                }
                __stcs(&n4[w], make_float4(nb[0], nb[1], nb[2], nb[3]));
                const int64_t e = 4 * w;
#pragma unroll
                for (int k = 0; k < 4; ++k) blk[e + k] = (uint16_t)code[k];
            }
        }
        (void)code4;
        // tail elements (e1 not a multiple of 4)
        for (int64_t e = 4 * v1 + threadIdx.x; e < e1; e += TK_THREADS) {
            const double b = (double)base[e];
            const int code = rquant(q_ds((double)cur[e], b), rq);
            blk[e] = (uint16_t)code;
            J.new_base[e] = radvance(b, code, rq);
        }
        return;
    }
    if (J.bits == 16) {
        uint16_t* blk = (uint16_t*)(J.out + 20);  // 2-byte aligned (out is 256-byte aligned)
        for (int64_t e = r0 * J.dims + threadIdx.x; e < e1; e += TK_THREADS) {
            const double b = (double)base[e];
            const int code = rquant(q_ds((double)cur[e], b), rq);
            blk[e] = (uint16_t)code;
            if (J.new_base) J.new_base[e] = radvance(b, code, rq);
        }
    } else {
        uint8_t* blk = J.out + 20;
        for (int64_t e = r0 * J.dims + threadIdx.x; e < e1; e += TK_THREADS) {
            const double b = (double)base[e];
            const int code = rquant(q_ds((double)cur[e], b), rq);
            blk[e] = (uint8_t)code;
            if (J.new_base) J.new_base[e] = radvance(b, code, rq);
        }
    }
}

template <typename T>
__device__ __forceinline__ void emit_sparse(const Job& J, const QParams& rq, int64_t c, int64_t r0, int64_t r1) {
    const T* cur = (const T*)J.cur;
    const T* base = (const T*)J.base;
    const int dims = J.dims, cb = J.bits / 8;
    uint8_t* blk = J.out + 24;
    const uint64_t V = J.var_pre[J.nchunks];
    const bool copy_base = J.new_base && (const void*)J.new_base != J.base;
    if (!J.ck[c]) {  // no survivor: the baseline rows are unchanged
        if (copy_base)
            for (int64_t e = r0 * dims + threadIdx.x; e < r1 * dims; e += TK_THREADS) J.new_base[e] = (float)base[e];
        return;
    }
    __shared__ uint32_t s_keep[TK_CHUNK / 32];
    __shared__ uint32_t s_wpre[TK_CHUNK / 32];   // survivors before each bitmap word
    __shared__ uint32_t s_vpre[TK_CHUNK / 32];   // varint bytes before each word (within chunk)
    __shared__ int64_t s_wprev[TK_CHUNK / 32];   // last kept row before each word (global)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int it = 0; it < TK_ITEMS; ++it) {
        const int64_t row = r0 + it * TK_THREADS + threadIdx.x;
        bool keep = false;
        if (row < r1) {
            double rmax = 0.0;
            for (int d = 0; d < dims; ++d) {
                const int64_t e = row * dims + d;
                rmax = np_max(rmax, fabs(q_ds((double)cur[e], (double)base[e])));
            }
            keep = rmax >= J.gate;
            if (!keep && copy_base)
                for (int d = 0; d < dims; ++d) J.new_base[row * dims + d] = (float)base[row * dims + d];
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_keep[it * (TK_THREADS / 32) + warp] = bal;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t k = J.cnt_pre[c];
        uint64_t v = 0;
        int64_t prev = J.prev_last[c];
        for (int w = 0; w < TK_CHUNK / 32; ++w) {
            s_wpre[w] = k;
            s_vpre[w] = (uint32_t)v;
            s_wprev[w] = prev;
            uint32_t bits = s_keep[w];
            k += __popc(bits);
            while (bits) {
                const int b = __ffs(bits) - 1;
                bits &= bits - 1;
                const int64_t row = r0 + 32 * w + b;
                v += vlen((uint64_t)(row - prev - 1));
                prev = row;
            }
        }
    }
    __syncthreads();
    const int w = threadIdx.x;
    if (w < TK_CHUNK / 32 && s_keep[w]) {
        uint32_t bits = s_keep[w];
        uint32_t k = s_wpre[w];
        uint64_t vo = J.var_pre[c] + s_vpre[w];
        int64_t prev = s_wprev[w];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int64_t row = r0 + 32 * w + b;
            const uint64_t gap = (uint64_t)(row - prev - 1);
            vput(blk + vo, gap);
            vo += vlen(gap);
            prev = row;
            uint8_t* cp = blk + V + (uint64_t)k * dims * cb;
            for (int d = 0; d < dims; ++d) {
                const int64_t e = row * dims + d;
                const double bb = (double)base[e];
                const uint32_t code = (uint32_t)rquant(q_ds((double)cur[e], bb), rq);
                if (cb == 2) {
                    cp[2 * d] = code & 0xff;
                    cp[2 * d + 1] = code >> 8;
                } else {
                    cp[d] = (uint8_t)code;
                }
                if (J.new_base) J.new_base[e] = radvance(bb, (int)code, rq);
            }
            ++k;
        }
    }
}

// One launch = [emit blocks of one residual job] + [scan blocks of the next
// residual job, or of every absolute job].  The emit part reads the plan the
// previous launch's last scan block wrote.

__device__ __forceinline__ void emit_chunk(const Job& J, int64_t c) {
    const int64_t r0 = c * TK_CHUNK;
    const int64_t r1 = min(r0 + TK_CHUNK, J.rows);
    const QParams rq = *J.rq;
    if (*J.mode == 0) {
        if (J.f64) emit_dense<double>(J, rq, r0, r1);
        else emit_dense<float>(J, rq, r0, r1);
    } else {
        if (J.f64) emit_sparse<double>(J, rq, c, r0, r1);
        else emit_sparse<float>(J, rq, c, r0, r1);
    }
}

__device__ __forceinline__ void scan_chunk(const Job& J, int64_t c) {
    const int64_t r0 = c * TK_CHUNK;
    const int64_t r1 = min(r0 + TK_CHUNK, J.rows);
    if (J.residual) {
        if (J.f64) scan_residual<double>(J, c, r0, r1);
        else scan_residual<float>(J, c, r0, r1);
        // the last block to finish this job's scan plans it
        __shared__ int s_last;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            s_last = atomicAdd(&J.g[3], 1ull) == (unsigned long long)(J.nchunks - 1);
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            plan_job(J);
        }
        return;
    }
    __shared__ int s_col[TK_MAX_DIMS];
    build_cols(J, s_col);
    if (J.f64) scan_absolute<double>(J, s_col, r0, r1);
    else scan_absolute<float>(J, s_col, r0, r1);
    if (c == 0 && threadIdx.x == 0) {
        const uint64_t blen = J.attr == 6 ? (uint64_t)(J.rows + 7) / 8 : (uint64_t)(J.rows * J.dims * J.bits + 7) / 8;
        uint8_t* o = J.out;
        o[0] = (uint8_t)J.attr;
        o[1] = 2;
        o[2] = 0;
        o[3] = (uint8_t)J.dims;
        put32(o + 4, (uint32_t)J.rows);
        put32(o + 8, (uint32_t)blen);
        *J.out_len = 12 + blen;
    }
}

#ifndef TK_EMIT_MINB
#define TK_EMIT_MINB 5  // <= 51 registers: 5 blocks per SM (measured dense tick 3/4/5/6 blocks: 76.8/74.7/72.7/80.9 us)
#endif
// one launch: [residual scans][absolute jobs][residual emits]; the emit
// blocks are dispatched after every scan block and wait on their job's plan
// flag (the absolute jobs in between cover the plan tail)
#ifndef TK_ORDER
#define TK_ORDER 0  // 0: [scans][absolute][emits]; 1: [scans][emits][absolute] (measured slower: 82.9 vs 78.8 us)
#endif
__global__ void __launch_bounds__(TK_THREADS, TK_EMIT_MINB) k_tick_fused(Batch B, int64_t res_chunks, int64_t abs_chunks,
                                                                          unsigned* __restrict__ ticket) {
    SS_PDL_WAIT();
    __shared__ unsigned s_ticket;
    if (threadIdx.x == 0) s_ticket = atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t b = s_ticket;
    // global chunk ids: residual jobs [0, res_chunks), absolute [res_chunks, res_chunks + abs_chunks)
    int64_t scan = -1, emit = -1;
    if (b < res_chunks) scan = b;
    else if (TK_ORDER == 1 && b < 2 * res_chunks) emit = b - res_chunks;
    else if (TK_ORDER == 1) scan = b - res_chunks;  // absolute chunk res_chunks + (b - 2 res_chunks)
    else if (b < res_chunks + abs_chunks) scan = b;
    else emit = b - res_chunks - abs_chunks;
    SS_ASSERT(b < 2 * res_chunks + abs_chunks);
    if (scan >= 0) {
        const Job& J = B.j[find_job(B, scan)];
        SS_ASSERT(scan - J.chunk0 >= 0 && scan - J.chunk0 < J.nchunks);
        scan_chunk(J, scan - J.chunk0);
        return;
    }
    const Job& J = B.j[find_job(B, emit)];
    SS_ASSERT(J.residual && emit - J.chunk0 >= 0 && emit - J.chunk0 < J.nchunks);
    wait_planned(J);
    emit_chunk(J, emit - J.chunk0);
}

}  // namespace

extern "C" int ss_encode_delta_batch(ss_ctx* ctx, const ss_delta_job* jobs, int32_t njobs) {
    SS_NVTX("ss_encode_delta_batch");
    if (!ctx || !jobs) return SS_ERR_INVALID;
    if (njobs < 1 || njobs > TK_MAX_JOBS) return ss_fail(ctx, SS_ERR_INVALID, "1..%d jobs per batch", TK_MAX_JOBS);
    SS_TRY(ss_scratch_reset(ctx));
    Batch B;
    memset(&B, 0, sizeof(B));
    B.n = njobs;
    int64_t chunks = 0;
    bool any_resid = false;
    size_t scratch = 0;
    for (int i = 0; i < njobs; ++i) {
        const ss_delta_job& s = jobs[i];
        Job& J = B.j[i];
        if (s.attribute_id < 0 || s.attribute_id > 6) return ss_fail(ctx, SS_ERR_PROTOCOL, "unknown attribute id %d", s.attribute_id);
        if (s.rows < 0 || s.dims < 1 || s.dims > TK_MAX_DIMS || s.rows > (int64_t)UINT32_MAX)
            return ss_fail(ctx, SS_ERR_INVALID, "bad delta shape");
        J.attr = s.attribute_id;
        J.residual = s.attribute_id <= 1;
        if (J.residual && (s.row_stride && s.row_stride != s.dims || s.inner && s.inner != s.dims || s.col0))
            return ss_fail(ctx, SS_ERR_INVALID, "residual deltas need contiguous (rows, dims) inputs");
        if (J.residual && !s.base && s.rows > 0)
            return ss_fail(ctx, SS_ERR_INVALID, "attribute %d is residual-coded and needs a baseline", J.attr);
        const int bits_tab[7] = {16, 8, 10, 8, 8, 8, 1};
        const double lo_tab[7] = {0, -10.0, -1.0, -8.0, -4.0, -1.0, 0.0};
        const double hi_tab[7] = {0, 2.0, 1.0, 8.0, 4.0, 1.0, 1.0};
        J.bits = bits_tab[J.attr];
        J.qlo = lo_tab[J.attr];
        J.qhi = hi_tab[J.attr];
        J.q = make_q(J.qlo, J.qhi, J.bits);
        if (J.bits == 10 && s.dims % 4) return ss_fail(ctx, SS_ERR_INVALID, "10-bit pack needs dims % 4 == 0");
        if (J.attr == 6 && s.dims != 1) return ss_fail(ctx, SS_ERR_INVALID, "visibility deltas have dims 1");
        if (s.out_cap < ss_delta_bound(J.attr, s.rows, s.dims)) return ss_fail(ctx, SS_ERR_CAPACITY, "delta output too small");
        J.cur = s.cur;
        J.base = s.base;
        J.new_base = s.new_base;
        J.out = s.out;
        J.out_len = s.out_len;
        J.rows = s.rows;
        J.dims = s.dims;
        J.row_stride = s.row_stride ? s.row_stride : s.dims;
        J.inner = s.inner ? s.inner : s.dims;
        J.outer = s.outer;
        J.col0 = s.col0;
        J.f64 = s.in_dtype == 1;
        J.gate = s.gating_threshold;
        if (!(J.gate > 1e-30)) {  // gate <= 0: rmax >= 0 >= gate keeps every row; tiny or NaN gates take the exact test
            J.gate_hi = J.gate <= 0.0 ? -1.0f : INFINITY;
            J.gate_lo = J.gate <= 0.0 ? -2.0f : -INFINITY;
        } else {
            J.gate_hi = nextafterf((float)(J.gate * (1.0 + 0x1p-20)), INFINITY);
            J.gate_lo = nextafterf((float)(J.gate * (1.0 - 0x1p-20)), -INFINITY);
        }
        J.nchunks = (s.rows + TK_CHUNK - 1) / TK_CHUNK;
        if (J.residual) any_resid = true;
    }
    // residual jobs' chunks first, absolute after: launch 1 runs the residual
    // scans and then the absolute jobs, whose streaming overlaps the plan tail
    for (int pass = 0; pass < 2; ++pass)
        for (int i = 0; i < njobs; ++i) {
            Job& J = B.j[i];
            if (J.residual != 1 - pass) continue;
            J.chunk0 = chunks;
            chunks += J.nchunks;
        }
    for (int i = 0; i < njobs; ++i) {
        Job& J = B.j[i];
        if (!J.residual) continue;
        const int64_t nc = J.nchunks + 1;
        J.g = SS_SCRATCH(ctx, unsigned long long, 4);
        J.ck = SS_SCRATCH(ctx, uint32_t, nc);
        J.cfirst = SS_SCRATCH(ctx, int64_t, nc);
        J.clast = SS_SCRATCH(ctx, int64_t, nc);
        J.cvar = SS_SCRATCH(ctx, uint32_t, nc);
        J.cmax = SS_SCRATCH(ctx, uint32_t, 2 * nc);
        J.cnt_pre = SS_SCRATCH(ctx, uint32_t, nc);
        J.var_pre = SS_SCRATCH(ctx, uint64_t, nc);
        J.prev_last = SS_SCRATCH(ctx, int64_t, nc);
        J.m = SS_SCRATCH(ctx, double, 1);
        J.rq = SS_SCRATCH(ctx, QParams, 1);
        J.mode = SS_SCRATCH(ctx, int, 1);
        if (!J.g || !J.ck || !J.cfirst || !J.clast || !J.cvar || !J.cmax || !J.cnt_pre || !J.var_pre || !J.prev_last || !J.m || !J.rq ||
            !J.mode)
            return SS_ERR_CUDA;
        SS_CUDA(ctx, cudaMemsetAsync(J.g, 0, 4 * sizeof(unsigned long long), ctx->stream));
        scratch += 1;
    }
    ss_tic(ctx, KC_CODEC);
    // one launch: [scan of every residual job (each job's last block plans
    // it)][every absolute job][emit of every residual job]; the emit re-reads
    // the residual inputs (24 B/row), partly from L2
    int64_t abs_chunks = 0, res_chunks = 0;
    for (int i = 0; i < njobs; ++i) (B.j[i].residual ? res_chunks : abs_chunks) += B.j[i].nchunks;
    for (int i = 0; i < njobs; ++i)
        if (B.j[i].residual && B.j[i].nchunks == 0) {  // no scan block: plan it here
            SS_CUDA(ctx, ss_launch((k_tick_plan), dim3(1), dim3(TK_THREADS), 0, ctx->stream, B, i));
            SS_CHECK_LAUNCH(ctx);
        }
    if (res_chunks + abs_chunks) {  // residual chunks are [0, res), absolute [res, res + abs)
        unsigned* ticket = SS_SCRATCH(ctx, unsigned, 1);
        if (!ticket) return SS_ERR_CUDA;
        SS_CUDA(ctx, cudaMemsetAsync(ticket, 0, sizeof(unsigned), ctx->stream));
        SS_CUDA(ctx, ss_launch((k_tick_fused), dim3((unsigned)(2 * res_chunks + abs_chunks)), dim3(TK_THREADS), 0, ctx->stream, B,
                               res_chunks, abs_chunks, ticket));
        SS_CHECK_LAUNCH(ctx);
    }
    // jobs with zero rows and no chunk still need their header
    for (int i = 0; i < njobs; ++i)
        if (B.j[i].rows == 0 && !B.j[i].residual) {
            SS_CUDA(ctx, ss_launch((k_empty_header), dim3(1), dim3(1), 0, ctx->stream, B, i));
            SS_CHECK_LAUNCH(ctx);
        }
    ss_toc(ctx, KC_CODEC);
    return SS_OK;
}
