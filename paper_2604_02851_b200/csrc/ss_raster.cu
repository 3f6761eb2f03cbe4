// Differentiable tile rasterizer for the splatstream compositing rules.
//
//   K1  k_preprocess    per Gaussian: fp64 projection, Sigma2d, 3-sigma
//                       window, depth key, relit colour     (render.py:226-290)
//   K3a depth sort      stable radix sort of fp64-depth bits -> exact
//                       lexsort((rows, depth)) order         (render.py:283)
//   K2  k_count/k_emit_warp rank-ordered splat records, tile-overlap counts,
//                       exclusive scan, (tile, rank) pair emission
//   K3b tile sort       stable radix sort on ceil(log2 tiles) key bits
//   K4  k_ranges        per-tile [start, end)
//   K5  k_blend_fwd     1 CTA per 16x16 tile; front-to-back with the
//                       reference's rules: rectangular window, T-gate
//                       before the splat, alpha cap 0.999, no 1/255 skip,
//                       CTA-wide early exit                 (render.py:304-336)
//   K6  k_blend_bwd     front-to-back again, S = C - prefix - contrib;
//                       4 pixels per thread, transposed warp reduction,
//                       one partial per (tile, splat) pair (deterministic)
//                                                            (optim.py:133-172)
//   K7  k_chain         per Gaussian: fixed-order sum of its partials and
//                       the chain rule to the 5 parameter groups, += into
//                       the flat gradient buffer          (optim.py:174-267)
//
// Precision: windows/depth always fp64; blending in fp32 (precision 0) or
// fp64 (precision 1).
#include "ss_project.cuh"

namespace {

constexpr int TILE = 16;
constexpr double T_CUTOFF = 1e-4;
constexpr double ALPHA_CAP = 0.999;

template <typename R>
struct __align__(16) SplatRec {
    int win[4];     // x0, x1, y0, y1 (first: 16-byte aligned for vector loads)
    R a, b, c;      // inverse 2D covariance [[a, b], [b, c]]
    R o;            // opacity
    R col[3];       // clamped colour
};



struct Bins {
    int64_t n_in;            // rows considered (subset or all)
    int64_t visible;
    int64_t pairs;
    int tiles_x, tiles_y, n_tiles, tile_bits;
    uint64_t* dkey64;        // [n_in] exact depth key (fp64 bits, ~0 = culled), by input index j
    uint32_t* dkeys;         // [n_in] 32-bit depth keys, sorted (0xffffffff = culled)
    uint32_t* dvals;         // [n_in] input index j, sorted by depth
    double2* mu;             // [n_in] fp64 centre, by input index j
    uint64_t* roff;          // [n_in] rank -> first pair (pre-sort position)
    uint32_t* rcnt;          // [n_in] tiles touched
    uint32_t* rinv;          // [n_in] input index j -> depth rank (~0 if culled)
    void* rec;               // [n_in] SplatRec<R>, by input index j
    uint64_t* roffj;         // [n_in] first pair of input j (= roff[rank(j)])
    uint32_t* pkeys;         // [pairs] tile id (sorted)
    uint32_t* pvals;         // [pairs] input index j of the splat (sorted by (tile, depth rank))
    uint2* ranges;           // [n_tiles]
    uint64_t* n_pairs;       // [1] device: pairs emitted (<= pairs, the host-side capacity)
};

// ---------------------------------------------------------------- K1
struct DebugOut {
    ss_prepared p;
    const uint64_t* vpos;    // visible position of input j
};

// the parameter columns of a model stored as PT (float; double for the
// fp64 instantiation's float64 models, ss_model.param_dtype = 1)
template <typename PT>
struct ParamView {
    const PT *means, *ls, *quats, *logit, *sh, *vis;
    __device__ __forceinline__ explicit ParamView(const ss_model& m)
        : means((const PT*)m.means), ls((const PT*)m.log_scales), quats((const PT*)m.quaternions),
          logit((const PT*)m.logit_opacities), sh((const PT*)m.sh_coeffs), vis((const PT*)m.light_visibility) {}
};

template <typename PT>
__global__ void k_visible_flags(ss_model m, ss_camera cam, const int64_t* subset, int64_t n_in, uint8_t* flag) {
    SS_PDL_WAIT();
    const ParamView<PT> pv(m);
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_in; j += (int64_t)gridDim.x * blockDim.x) {
        int64_t row = subset ? subset[j] : j;
        double d[3], mc[3];
        ss_cam_point(cam, pv.means + row * 3, d, mc);
        flag[j] = mc[2] >= cam.near_plane;
    }
}

template <int DEG, typename R, typename PT>
#ifndef SS_PRE_MINB
#define SS_PRE_MINB 3  // with the up-front parameter loads (measured 3 / 4 / 5: 0.84 / 0.89 / 0.98 ms per step)
#endif
#ifndef SS_PRE_PREFETCH
#define SS_PRE_PREFETCH 1
#endif
__global__ void __launch_bounds__(128, SS_PRE_MINB) k_preprocess(ss_model m, ss_camera cam, ss_light L, const int64_t* __restrict__ subset, int64_t n_in,
                             int cutoff, uint64_t* __restrict__ dkeys, uint32_t* __restrict__ dvals,
                             SplatRec<R>* __restrict__ rec, double2* __restrict__ mu, DebugOut dbg,
                             unsigned long long* __restrict__ kminmax) {
    SS_PDL_WAIT();
    unsigned long long kmin = ~0ull, kmax = 0;
    constexpr int B = ss_sh_bases(DEG);
    const ParamView<PT> pv(m);
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_in; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = subset ? subset[j] : j;
#if SS_PRE_PREFETCH
        // every parameter load of the row first (the stores below would otherwise hold them back)
        PT lsv[3], qv[4], shv[3 * B];
#pragma unroll
        for (int k = 0; k < 3; ++k) lsv[k] = pv.ls[row * 3 + k];
#pragma unroll
        for (int k = 0; k < 4; ++k) qv[k] = pv.quats[row * 4 + k];
        ss_load_sh<DEG, PT>(pv.sh + row * 3 * B, shv);
        const PT logit = pv.logit[row], visv = pv.vis[row];
#else
        const PT* lsv = pv.ls + row * 3;
        const PT* qv = pv.quats + row * 4;
#endif
        Proj P;
        ss_cam_point(cam, pv.means + row * 3, P.d, P.mc);
        dvals[j] = (uint32_t)j;
        if (!(P.mc[2] >= cam.near_plane)) {
            dkeys[j] = ~0ull;
            continue;
        }
        dkeys[j] = (uint64_t)__double_as_longlong(P.mc[2]);  // z >= near > 0: bits order as the value
        kmin = min(kmin, (unsigned long long)dkeys[j]);
        kmax = max(kmax, (unsigned long long)dkeys[j]);
        ss_project(cam, lsv, qv, cutoff != 0, P);
        Shade<DEG, R> S;
        {
#if !SS_PRE_PREFETCH
            PT shv[3 * B];
            ss_load_sh<DEG, PT>(pv.sh + row * 3 * B, shv);
            const PT visv = pv.vis[row];
#endif
            const R dR[3] = {(R)P.d[0], (R)P.d[1], (R)P.d[2]};
            R RqR[3][3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int k = 0; k < 3; ++k) RqR[i][k] = (R)P.Rq[i][k];
            ss_shade_v<DEG, R, PT>(L, lsv, shv, visv, dR, RqR, S);
        }
        SplatRec<R> g;
        g.a = (R)(P.s11 / P.det);
        g.b = (R)(-P.s01 / P.det);
        g.c = (R)(P.s00 / P.det);
#if !SS_PRE_PREFETCH
        const PT logit = pv.logit[row];
#endif
        g.o = sizeof(R) == 4 ? (R)(1.0f / (1.0f + expf(-(float)logit))) : (R)(1.0 / (1.0 + exp(-(double)logit)));
        for (int c = 0; c < 3; ++c) g.col[c] = (R)fmin(fmax((double)S.pre[c], 0.0), 1.0);
        ss_window(P, cam.width, cam.height, g.win);
        rec[j] = g;
        mu[j] = make_double2(P.mu[0], P.mu[1]);
        if (dbg.vpos) {
            const int64_t v = (int64_t)dbg.vpos[j];
            const ss_prepared& o = dbg.p;
            if (o.rows) o.rows[v] = row;
            if (o.depth) o.depth[v] = P.mc[2];
            if (o.mu2d) { o.mu2d[2 * v] = P.mu[0]; o.mu2d[2 * v + 1] = P.mu[1]; }
            if (o.sigma2d) { o.sigma2d[3 * v] = P.s00; o.sigma2d[3 * v + 1] = P.s01; o.sigma2d[3 * v + 2] = P.s11; }
            if (o.radius) o.radius[v] = P.radius;
            if (o.window) for (int k = 0; k < 4; ++k) o.window[4 * v + k] = g.win[k];
            if (o.opacity) o.opacity[v] = g.o;
            if (o.color) for (int c = 0; c < 3; ++c) o.color[3 * v + c] = g.col[c];
            if (o.color_pre) for (int c = 0; c < 3; ++c) o.color_pre[3 * v + c] = S.pre[c];
            if (o.shade_s) o.shade_s[v] = S.s;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmin, o), b = __shfl_xor_sync(0xffffffffu, kmax, o);
        kmin = min(kmin, a);
        kmax = max(kmax, b);
    }
    if ((threadIdx.x & 31) == 0 && kmin != ~0ull) {
        atomicMin(&kminmax[0], kmin);
        atomicMax(&kminmax[1], kmax);
    }
}

__global__ void k_init_minmax(unsigned long long* kminmax) {
    SS_PDL_WAIT();
    kminmax[0] = ~0ull;
    kminmax[1] = 0ull;
}

// 32-bit depth keys: the exact fp64-bit key minus the minimum, shifted so the
// range fits 32 bits.  The shift can merge nearly equal depths; k_fix_ties
// restores the exact order inside such runs.
__global__ void k_key32(const uint64_t* __restrict__ dkey64, int64_t n, const unsigned long long* __restrict__ kminmax,
                        uint32_t* __restrict__ key32) {
    SS_PDL_WAIT();
    const unsigned long long lo = kminmax[0], hi = kminmax[1];
    const unsigned long long range = hi > lo ? hi - lo : 0;
    const int bits = range ? 64 - __clzll((long long)range) : 0;
    const int shift = bits > 32 ? bits - 32 : 0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = dkey64[j];
        uint32_t v = 0xffffffffu;
        if (k != ~0ull) {
            const unsigned long long d = (k - lo) >> shift;
            v = d > 0xfffffffeull ? 0xfffffffeu : (uint32_t)d;
        }
        key32[j] = v;
    }
}

// Runs of equal 32-bit keys (rare: depths equal to ~2^-32 relative) are put
// in exact (depth, row) order by one thread each; the sort was stable, so a
// stable insertion sort on the exact key gives lexsort((rows, depth)).
__global__ void k_fix_ties(const uint32_t* __restrict__ key32, uint32_t* __restrict__ vals,
                           const uint64_t* __restrict__ dkey64, int64_t n) {
    SS_PDL_WAIT();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = key32[i];
        if (k == 0xffffffffu || key32[i + 1] != k || (i > 0 && key32[i - 1] == k)) continue;
        int64_t e = i + 1;
        while (e < n && key32[e] == k) ++e;
        for (int64_t a = i + 1; a < e; ++a) {
            const uint32_t v = vals[a];
            const uint64_t kv = dkey64[v];
            int64_t b = a - 1;
            while (b >= i && dkey64[vals[b]] > kv) {
                vals[b + 1] = vals[b];
                --b;
            }
            vals[b + 1] = v;
        }
    }
}

// ---------------------------------------------------------------- K2
__device__ __forceinline__ void win_tiles(const int w[4], int& tx0, int& tx1, int& ty0, int& ty1) {
    tx0 = w[0] / TILE;
    tx1 = (w[1] - 1) / TILE;
    ty0 = w[2] / TILE;
    ty1 = (w[3] - 1) / TILE;
}

template <typename R>
__global__ void k_count(const uint64_t* __restrict__ dkey64, const uint32_t* __restrict__ dvals,
                        const SplatRec<R>* __restrict__ rec, int64_t n_in, uint32_t* __restrict__ rcnt,
                        uint32_t* __restrict__ rinv) {
    SS_PDL_WAIT();
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_in; r += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t j = dvals[r];
        const uint64_t key = dkey64[j];
        const int4 w = *reinterpret_cast<const int4*>(rec[j].win);  // both loads before any store
        if (key == ~0ull) {
            rcnt[r] = 0;
            rinv[j] = ~0u;
            continue;
        }
        rinv[j] = (uint32_t)r;
        const int win[4] = {w.x, w.y, w.z, w.w};
        uint32_t cnt = 0;
        if (win[0] < win[1] && win[2] < win[3]) {
            int tx0, tx1, ty0, ty1;
            win_tiles(win, tx0, tx1, ty0, ty1);
            cnt = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
        }
        rcnt[r] = cnt;
    }
}

// Pair emission: every (tile, splat) pair, splats in rank order, a splat's
// tiles row-major from roff[rank].  A warp takes 32
// consecutive ranks, whose pairs form one contiguous output range, and writes
// that range 32 pairs at a time; each lane finds the rank owning its pair by
// a 5-step binary search over the lanes' start offsets (shuffles), so the
// stores are coalesced and a large splat no longer serialises one thread.
template <typename R>
__global__ void __launch_bounds__(256) k_emit_warp(const SplatRec<R>* __restrict__ rec, const uint32_t* __restrict__ dvals,
                                                   const uint32_t* __restrict__ rcnt, const uint64_t* __restrict__ roff,
                                                   int64_t n_in, int tiles_x, uint32_t* __restrict__ pkeys,
                                                   uint32_t* __restrict__ pvals, uint64_t* __restrict__ roffj,
                                                   uint64_t cap) {
    SS_PDL_WAIT();
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; r0 < n_in; r0 += nwarps * 32) {
        const int64_t r = r0 + lane;
        const uint32_t cnt = r < n_in ? rcnt[r] : 0u;
        const uint64_t off = r < n_in ? roff[r] : ~0ull;
        uint32_t j = 0;
        int tx0 = 0, ty0 = 0, w = 1;
        if (cnt) {
            j = dvals[r];
            int tx1, ty1;
            win_tiles(rec[j].win, tx0, tx1, ty0, ty1);
            w = tx1 - tx0 + 1;
            roffj[j] = off;
        }
        const uint64_t p0 = __shfl_sync(0xffffffffu, off, 0);
        uint64_t p1 = cnt ? off + cnt : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const uint64_t t = __shfl_xor_sync(0xffffffffu, p1, o);
            p1 = t > p1 ? t : p1;
        }
        for (uint64_t base = p0; base < p1; base += 32) {
            const uint64_t p = base + lane;
            int src = 0;  // the last lane whose range starts at or before p
#pragma unroll
            for (int step = 16; step; step >>= 1) {
                const uint64_t o = __shfl_sync(0xffffffffu, off, src + step);
                if (o <= p) src += step;
            }
            const uint64_t so = __shfl_sync(0xffffffffu, off, src);
            const uint32_t sj = __shfl_sync(0xffffffffu, j, src);
            const int sx = __shfl_sync(0xffffffffu, tx0, src), sy = __shfl_sync(0xffffffffu, ty0, src);
            const int sw = __shfl_sync(0xffffffffu, w, src);
            if (p < p1 && p < cap) {  // beyond the capacity: the call overflowed (flagged, results void)
                const uint32_t q = (uint32_t)(p - so);
                const uint32_t qy = q / (uint32_t)sw;
                SS_ASSERT(sj < (uint64_t)n_in && (int)(q - qy * (uint32_t)sw) < sw);
                pkeys[p] = (uint32_t)((sy + (int)qy) * tiles_x + sx + (int)(q - qy * (uint32_t)sw));
                pvals[p] = sj;
            }
        }
    }
}

__global__ void k_ranges(const uint32_t* __restrict__ keys, const uint64_t* __restrict__ n_dev, uint2* __restrict__ ranges) {
    SS_PDL_WAIT();
    const int64_t n = (int64_t)*n_dev;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t t = keys[s];
        SS_ASSERT(s == 0 || keys[s - 1] <= t);  // sorted by tile
        if (s == 0 || keys[s - 1] != t) ranges[t].x = (uint32_t)s;
        if (s == n - 1 || keys[s + 1] != t) ranges[t].y = (uint32_t)(s + 1);
    }
}

// ---------------------------------------------------------------- blend math
//
// One warp owns one 16x16 tile; lane l holds the 8 pixels (l % 16, l / 16 + 2q),
// q = 0..7.  A warp stages 32 splats at a time in shared memory and walks
// them in depth order; no block-level barriers anywhere (blocks are just
// WPB independent tiles).  Per-pixel liveness is an 8-bit mask; a pixel dies
// when T drops below 1e-4 (the reference's T-gate: later splats skip it).
#ifndef SS_WPB
#define SS_WPB 4
#endif
constexpr int WPB = SS_WPB;   // tiles (warps) per block of the forward kernels
#ifndef SS_WPB_BWD
#define SS_WPB_BWD 1  // measured (bench backward class per step): 1 / 2 / 4 -> 9.36 / 9.40 / 9.68 ms
#endif
constexpr int WPB_BWD = SS_WPB_BWD;  // ... of the backward (fewer tiles per block: less waiting on a block's slowest tile)
constexpr int PPT = 8;   // pixels per lane
// pixel rows per warp-uniform skip test: rows of one group form one basic
// block, so their independent chains interleave (helps the longer backward
// body; the short forward body prefers the finer skip)
constexpr int QG_FWD = 1, QG_BWD = 2;

template <typename R> __device__ __forceinline__ R ss_exp(R x);
template <> __device__ __forceinline__ float ss_exp<float>(float x) { return __expf(x); }
template <> __device__ __forceinline__ double ss_exp<double>(double x) { return exp(x); }

template <typename R> __device__ __forceinline__ R ss_rcp(R x);
template <> __device__ __forceinline__ float ss_rcp<float>(float x) {  // x = 1 - alpha >= 0.001
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float ss_ex2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
template <> __device__ __forceinline__ double ss_rcp<double>(double x) { return 1.0 / x; }
// alive &= ~bit when T < 1e-4 (the T-gate), as one predicated AND
__device__ __forceinline__ void gate_t(unsigned& alive, float t, unsigned bit) {
    asm("{\n .reg .pred p;\n setp.lt.f32 p, %1, 0f38D1B717;\n @p and.b32 %0, %0, %2;\n}\n"
        : "+r"(alive) : "f"(t), "r"(~bit));
}
__device__ __forceinline__ void gate_t(unsigned& alive, double t, unsigned bit) {
    if (t < T_CUTOFF) alive &= ~bit;
}

// Staged splat.  fp32: centre relative to the tile origin (rounded from the
// fp64 centre) so dx keeps full precision; fp64: absolute centre and
// dx = (px + 0.5) - mu exactly as the reference computes it.
template <typename R>
struct __align__(16) Staged {
    R mx, my, a, b;
    R c, o, c0, c1;
    R c2;
    R aK, bK2, cK;           // fp32: a K, 2 b K, c K with K = -0.5 log2(e) (the exponent's prescale), once per splat
    int wx;                  // tile-local x window: wx0 | (wx1 - wx0) << 16
    int rows;                // pixel-row masks of the y window: bits 0-7 even lanes, 8-15 odd lanes
    int p, pad;              // p = partial index (backward)
};

template <typename R>
__device__ __forceinline__ void stage(Staged<R>& s, const double2 mu, const SplatRec<R>& rec, int X0, int Y0) {
    if (sizeof(R) == 4) {
        s.mx = (R)(mu.x - (double)X0);
        s.my = (R)(mu.y - (double)Y0);
    } else {
        s.mx = (R)mu.x;
        s.my = (R)mu.y;
    }
    s.a = rec.a;
    s.b = rec.b;
    s.c = rec.c;
    s.o = rec.o;
    s.c0 = rec.col[0];
    s.c1 = rec.col[1];
    s.c2 = rec.col[2];
    if (sizeof(R) == 4) {
        const R K = (R)(-0.5 * 1.4426950408889634);
        s.aK = rec.a * K;
        s.bK2 = (R)2 * rec.b * K;
        s.cK = rec.c * K;
    }
    const int wx0 = min(max(rec.win[0] - X0, 0), TILE), wx1 = min(max(rec.win[1] - X0, 0), TILE);
    const int wy0 = min(max(rec.win[2] - Y0, 0), TILE), wy1 = min(max(rec.win[3] - Y0, 0), TILE);
    s.wx = wx0 | ((wx1 - wx0) << 16);
    unsigned rows = 0;
#pragma unroll
    for (int ly0 = 0; ly0 < 2; ++ly0) {  // rows ly0 + 2q inside [wy0, wy1), once per staged splat
        const int qlo = max(0, (wy0 - ly0 + 1) >> 1);
        const int qhi = max(0, (wy1 - ly0 + 1) >> 1);
        rows |= (((1u << qhi) - 1u) & ~((1u << qlo) - 1u)) << (8 * ly0);
    }
    s.rows = (int)rows;
}

// 8-bit mask of this lane's pixels (rows ly0 + 2q) inside the y window, if its column is inside the x window
template <typename R>
__device__ __forceinline__ unsigned lane_mask(const Staged<R>& s, int lx, int ly0) {
    if ((unsigned)(lx - (s.wx & 0xFFFF)) >= ((unsigned)s.wx >> 16)) return 0u;
    return ((unsigned)s.rows >> (8 * ly0)) & 0xFFu;
}

// the lane's pixel-centre coordinate: fp32 relative to the tile origin (the
// staged centre is too), fp64 absolute, (i + 0.5) as the reference (render.py:306-307)
template <typename R>
__device__ __forceinline__ R lane_centre(int l, int origin) {
    return sizeof(R) == 4 ? (R)l + (R)0.5 : (R)(origin + l) + (R)0.5;
}

template <typename R>
__device__ __forceinline__ R gauss_power(const Staged<R>& s, R dx, R dy) {
    return (R)-0.5 * (s.a * dx * dx + (R)2 * s.b * dx * dy + s.c * dy * dy);
}

// Per (splat, lane) geometry: the lane's column is fixed, so the conic's x
// terms are hoisted; per pixel the exponent is two FMAs.  fp64 keeps the
// reference's exact expression (render.py:311).
template <typename R, bool STAGED_K = false>
struct PixelGeom {
    // fp32: exponent pre-scaled by K = -0.5 log2(e) so G = ex2((cK y + BK) y + AK);
    // STAGED_K: the prescaled conic comes from the staging (forward)
    R dx, dy0, Ax2, Bx2, adx0, bdx0, cK;
    // (pxc, pyc): the lane's first pixel centre (tile-relative for fp32,
    // absolute for fp64), computed once per kernel by lane_centre
    __device__ __forceinline__ PixelGeom(const Staged<R>& s, R pxc, R pyc) {
        dx = pxc - s.mx;
        dy0 = pyc - s.my;
        adx0 = s.a * dx;
        bdx0 = s.b * dx;
        if (sizeof(R) == 4 && STAGED_K) {
            Ax2 = s.aK * dx * dx;
            Bx2 = s.bK2 * dx;
            cK = s.cK;
        } else if (sizeof(R) == 4) {
            const R K = (R)(-0.5 * 1.4426950408889634);
            Ax2 = adx0 * dx * K;
            Bx2 = (R)2 * bdx0 * K;
            cK = s.c * K;
        } else {
            Ax2 = s.a * dx * dx;
            Bx2 = (R)2 * s.b * dx;
            cK = s.c;
        }
    }
    __device__ __forceinline__ R dy(int q) const { return dy0 + (R)(2 * q); }
    __device__ __forceinline__ R gauss(const Staged<R>& s, int q) const {
        const R y = dy(q);
        if constexpr (sizeof(R) == 4) return ss_ex2((cK * y + Bx2) * y + Ax2);
        else return ss_exp<R>(gauss_power(s, dx, y));
    }
};

// ---------------------------------------------------------------- K5 forward
template <typename R>
__global__ void __launch_bounds__(32 * WPB) k_blend_fwd(const uint2* __restrict__ ranges,
                                                        const uint32_t* __restrict__ pvals,
                                                        const double2* __restrict__ mu,
                                                        const SplatRec<R>* __restrict__ rec, int W, int H,
                                                        int tiles_x, int n_tiles, double bg0, double bg1, double bg2,
                                                        R* __restrict__ img, R* __restrict__ Tout,
                                                        uint32_t* __restrict__ tile_stop,
                                                        unsigned long long* __restrict__ eval_count,
                                                        const uint32_t* __restrict__ order) {
    SS_PDL_WAIT();
    __shared__ Staged<R> sm[WPB][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = blockIdx.x * WPB + warp;
    if (slot >= n_tiles) return;
    const int tile = order ? (int)order[slot] : slot;
    const int X0 = (tile % tiles_x) * TILE, Y0 = (tile / tiles_x) * TILE;
    const int lx = lane & 15, ly0 = lane >> 4;
    const R pxc = lane_centre<R>(lx, X0), pyc = lane_centre<R>(ly0, Y0);
    unsigned alive = 0;
#pragma unroll
    for (int q = 0; q < PPT; ++q)
        if (X0 + lx < W && Y0 + ly0 + 2 * q < H) alive |= 1u << q;
    R T[PPT], C0[PPT], C1[PPT], C2[PPT];
#pragma unroll
    for (int q = 0; q < PPT; ++q) T[q] = 1, C0[q] = 0, C1[q] = 0, C2[q] = 0;
    const uint2 rg = ranges[tile];
    int last = -1;
    uint32_t evals = 0;
    Staged<R>* my = sm[warp];
    for (uint32_t b0 = rg.x; b0 < rg.y; b0 += 32) {
        if (!__any_sync(0xffffffffu, alive)) break;
        const uint32_t i = b0 + lane;
        if (i < rg.y) {
            const uint32_t j = pvals[i];
            stage(my[lane], mu[j], rec[j], X0, Y0);
        }
        __syncwarp();
        const int nb = (int)min(32u, rg.y - b0);
        for (int k = 0; k < nb; ++k) {
            const Staged<R> s = my[k];
            const unsigned act = lane_mask(s, lx, ly0) & alive;
            if (!act) continue;
            last = (int)(b0 - rg.x) + k;
            evals += __popc(act);
            // branch-free over the lane's 8 pixels: inactive ones get G = 0,
            // which leaves C and T unchanged
            PixelGeom<R> pg(s, pxc, pyc);
            const unsigned wact = __reduce_or_sync(__activemask(), act);
#pragma unroll
            for (int g = 0; g < PPT; g += QG_FWD) {
                if (!((wact >> g) & ((1u << QG_FWD) - 1u))) continue;  // warp-uniform: no lane needs these rows
#pragma unroll
                for (int q = g; q < g + QG_FWD; ++q) {
                    const R G = (act >> q) & 1u ? pg.gauss(s, q) : (R)0;
                    const R alpha = min(s.o * G, (R)ALPHA_CAP);
                    const R w = alpha * T[q];
                    C0[q] += w * s.c0;
                    C1[q] += w * s.c1;
                    C2[q] += w * s.c2;
                    T[q] -= w;  // T (1 - alpha)
                    gate_t(alive, T[q], 1u << q);
                }
            }
        }
        __syncwarp();
    }
    last = __reduce_max_sync(0xffffffffu, last + 1);
    if (lane == 0 && tile_stop) tile_stop[tile] = (uint32_t)last;
    if (eval_count) {
        evals = __reduce_add_sync(0xffffffffu, evals);
        if (lane == 0 && evals) atomicAdd(eval_count, (unsigned long long)evals);
    }
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
        const int px = X0 + lx, py = Y0 + ly0 + 2 * q;
        if (px < W && py < H) {
            const int64_t p = (int64_t)py * W + px;
            img[3 * p + 0] = C0[q] + T[q] * (R)bg0;
            img[3 * p + 1] = C1[q] + T[q] * (R)bg1;
            img[3 * p + 2] = C2[q] + T[q] * (R)bg2;
            if (Tout) Tout[p] = T[q];
        }
    }
}

// ---------------------------------------------------------------- K6 backward
// the colour clamp's gradient mask from the forward's clamped colour:
// col = clamp(color_pre, 0, 1) lies strictly inside (0, 1) exactly when
// color_pre does (ref optim.py:176-177)
template <typename R>
__device__ __forceinline__ bool clamp_open(R col) { return col > (R)0 && col < (R)1; }

// Transposed butterfly: reduces v[0..7] over the warp with 7+2 shuffles;
// lane l with (l & 3) == 0 ends with the sum of value index
// 4*bit4(l) + 2*bit3(l) + bit2(l).
template <typename R>
__device__ __forceinline__ R warp_reduce8(const R v[8], int lane) {
    R w[4];
    {
        const bool hi = lane & 16;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            R send = hi ? v[i] : v[i + 4];
            R keep = hi ? v[i + 4] : v[i];
            w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
    }
    R x[2];
    {
        const bool hi = lane & 8;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            R send = hi ? w[i] : w[i + 2];
            R keep = hi ? w[i + 2] : w[i];
            x[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
    }
    const bool hi = lane & 4;
    R y = (hi ? x[1] : x[0]) + __shfl_xor_sync(0xffffffffu, hi ? x[0] : x[1], 4);
    y += __shfl_xor_sync(0xffffffffu, y, 2);
    y += __shfl_xor_sync(0xffffffffu, y, 1);
    return y;
}

template <typename R>
__device__ __forceinline__ R warp_sum(R v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ uint32_t pair_index(const uint64_t* roff, const int win[4], uint32_t r, int tx, int ty) {
    int tx0, tx1, ty0, ty1;
    win_tiles(win, tx0, tx1, ty0, ty1);
    return (uint32_t)(roff[r] + (uint64_t)((ty - ty0) * (tx1 - tx0 + 1) + (tx - tx0)));
}

#ifdef SS_BWD_STATS
// utilisation counters of the backward walk (diagnostics build only):
// [0] pairs in the lists, [1] pairs walked, [2] walked pairs with an active
// pixel, [3] active (pixel, splat) pairs, [4] lanes entering the body,
// [5] pixel slots computed (executed row groups x QG x body lanes)
__device__ unsigned long long g_bwd_stats[8];
#endif
// ATOMIC (the throughput mode, ss_render_opts.deterministic = 0): each
// (tile, splat) pair's 9 warp-reduced sums are added straight into the
// splat's screen-space record g9[j] with float atomics (no partials, no
// k_sum_partials pass); the order of the additions across tiles is the
// scheduler's, so reruns can differ in the last bits.  Otherwise one partial
// per pair, summed in a fixed order by k_sum_partials (deterministic).
// blocks (tiles) per SM asked of the register allocation: 24 -> 80 registers.
// The kernel alone is 0.7 % slower than at its own best (96 registers), but
// the step is 1 % faster: the freed registers host the other lanes' kernels
// (measured, 8-view step: unbounded / 20 / 22 / 24 / 26 / 28 / 32 ->
// 473.4 / 474.5 / 476.7 / 478.6 / 474.7 / 473.0 / 465.9 views/s)
#ifndef SS_BWD_MINB
#define SS_BWD_MINB 24
#endif
#if SS_BWD_MINB > 0
#define SS_BWD_BOUNDS __launch_bounds__(32 * WPB_BWD, SS_BWD_MINB)
#else
#define SS_BWD_BOUNDS __launch_bounds__(32 * WPB_BWD)
#endif
template <typename R, bool ATOMIC = false>
__global__ void SS_BWD_BOUNDS k_blend_bwd(const uint2* __restrict__ ranges,
                                                        const uint32_t* __restrict__ pvals,
                                                        const double2* __restrict__ mu,
                                                        const SplatRec<R>* __restrict__ rec_,
                                                        const uint64_t* __restrict__ roffj,
                                                        const uint32_t* __restrict__ tile_stop, int W, int H,
                                                        int tiles_x, int n_tiles, const R* __restrict__ img,
                                                        const float* __restrict__ gt, double npx3,
                                                        R* __restrict__ partials, double* __restrict__ tile_loss,
                                                        const uint32_t* __restrict__ order, uint64_t cap) {
    SS_PDL_WAIT();
    __shared__ Staged<R> sm[WPB_BWD][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = blockIdx.x * WPB_BWD + warp;
    if (slot >= n_tiles) return;
    const int tile = order ? (int)order[slot] : slot;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int X0 = tx * TILE, Y0 = ty * TILE;
    const int lx = lane & 15, ly0 = lane >> 4;
    const R pxc = lane_centre<R>(lx, X0), pyc = lane_centre<R>(ly0, Y0);
    const uint2 rg = ranges[tile];
    const uint32_t stop = rg.x + (tile_stop ? min(tile_stop[tile], rg.y - rg.x) : (rg.y - rg.x));

    // per pixel: T, R = sum_c gC_c (C_c - prefix_c), dL/dC (gC), alive bit
    R T[PPT], Rr[PPT], g0[PPT], g1[PPT], g2[PPT];
    unsigned alive = 0;
    double loss = 0.0;
    const R inv = sizeof(R) == 8 ? (R)0 : (R)(1.0 / npx3);
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
        const int px = X0 + lx, py = Y0 + ly0 + 2 * q;
        T[q] = 1;
        Rr[q] = 0;
        g0[q] = g1[q] = g2[q] = 0;
        if (px < W && py < H) {
            alive |= 1u << q;
            const int64_t p = (int64_t)py * W + px;
            R gg[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const R v = img[3 * p + c];
                const R diff = v - (R)gt[3 * p + c];
                loss += fabs((double)diff);
                const R sg = diff > (R)0 ? (R)1 : (diff < (R)0 ? (R)-1 : (R)0);
                // dL/dC = sign(C - gt) / (H W 3)  (optim.py:124-125)
                gg[c] = sizeof(R) == 8 ? (R)((double)sg / npx3) : sg * inv;
                Rr[q] += gg[c] * v;
            }
            g0[q] = gg[0];
            g1[q] = gg[1];
            g2[q] = gg[2];
        }
    }
    Staged<R>* my = sm[warp];
#ifdef SS_BWD_STATS
    unsigned long long st[6] = {rg.y - rg.x, stop - rg.x, 0, 0, 0, 0};
#endif
    for (uint32_t b0 = rg.x; b0 < stop; b0 += 32) {
        const uint32_t i = b0 + lane;
        if (i < stop) {
            const uint32_t j = pvals[i];
            SS_ASSERT(i < rg.y && (uint64_t)i < cap);
            const SplatRec<R> rec = rec_[j];
            stage(my[lane], mu[j], rec, X0, Y0);
            my[lane].p = ATOMIC ? (int)j : (int)pair_index(roffj, rec.win, j, tx, ty);
        }
        __syncwarp();
        const int nb = (int)min(32u, stop - b0);
        for (int k = 0; k < nb; ++k) {
            const Staged<R> s = my[k];
            const unsigned act = lane_mask(s, lx, ly0) & alive;
            R acc[9];
#pragma unroll
            for (int e = 0; e < 9; ++e) acc[e] = 0;
#ifdef SS_BWD_STATS
            {
                const unsigned body = __ballot_sync(0xffffffffu, act != 0);
                const unsigned wa = __reduce_or_sync(0xffffffffu, act);
                int groups = 0;
                for (int g = 0; g < PPT; g += QG_BWD) groups += ((wa >> g) & ((1u << QG_BWD) - 1u)) ? 1 : 0;
                st[2] += body ? 1 : 0;
                st[3] += __reduce_add_sync(0xffffffffu, __popc(act));
                st[4] += __popc(body);
                st[5] += (unsigned long long)groups * QG_BWD * __popc(body);
            }
#endif
            if (act) {
                // branch-free over the lane's 8 pixels: inactive ones get
                // G = 0, which zeroes every contribution and leaves T, R alone
                PixelGeom<R, true> pg(s, pxc, pyc);
                const unsigned wact = __reduce_or_sync(__activemask(), act);
#pragma unroll
                for (int g = 0; g < PPT; g += QG_BWD) {
                    if (!((wact >> g) & ((1u << QG_BWD) - 1u))) continue;  // warp-uniform skip
#pragma unroll
                    for (int q = g; q < g + QG_BWD; ++q) {
                        const R G = (act >> q) & 1u ? pg.gauss(s, q) : (R)0;
                        const R oG = s.o * G;
                        const bool open = oG < (R)ALPHA_CAP;
                        const R alpha = open ? oG : (R)ALPHA_CAP;
                        const R w = alpha * T[q];
                        const R gcol = g0[q] * s.c0 + g1[q] * s.c1 + g2[q] * s.c2;
                        acc[0] += g0[q] * w;
                        acc[1] += g1[q] * w;
                        acc[2] += g2[q] * w;
                        // dL/dalpha = sum_c gC_c (col_c T - S_c / (1 - alpha)), S = C - prefix - contrib
                        const R rest = Rr[q] - w * gcol;
                        const R dal = T[q] * gcol - rest * ss_rcp<R>((R)1 - alpha);
                        Rr[q] = rest;
                        const R dalm = open ? dal : (R)0;  // capped alpha: no gradient
                        const R dG = dalm * G;
                        const R gp = dalm * alpha;
                        const R y = pg.dy(q);
                        const R adx = pg.adx0 + s.b * y;
                        const R ady = pg.bdx0 + s.c * y;
                        const R gpx = gp * adx, gpy = gp * ady;
                        acc[3] += dG;
                        acc[4] += gpx;
                        acc[5] += gpy;
                        acc[6] += gpx * adx;
                        acc[7] += gpx * ady;
                        acc[8] += gpy * ady;
                        T[q] -= w;
                        if (T[q] < (R)T_CUTOFF) alive &= ~(1u << q);
                    }
                }
            }
            R* out = partials + (uint64_t)(uint32_t)s.p * 9;
            const bool fits = ATOMIC || (uint64_t)(uint32_t)s.p < cap;  // else an overflowed call (flagged)
            if (__any_sync(0xffffffffu, act != 0)) {
                const R y = warp_reduce8<R>(acc, lane);
                const R z = warp_sum<R>(acc[8]);
                if ((lane & 3) == 0 && fits) {
                    const int e = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
                    R v = e >= 6 ? (R)0.5 * y : y;
                    if (ATOMIC) {  // no partial-sum pass: the clamp mask here
                        if (e < 3 && !clamp_open(e == 0 ? s.c0 : (e == 1 ? s.c1 : s.c2))) v = (R)0;
                        atomicAdd(out + e, v);
                    } else {
                        out[e] = v;
                    }
                }
                if (lane == 0 && fits) {
                    if (ATOMIC) atomicAdd(out + 8, (R)0.5 * z);
                    else out[8] = (R)0.5 * z;
                }
            } else if (!ATOMIC && lane < 9 && fits) {
                out[lane] = 0;
            }
        }
        __syncwarp();
    }
    // pairs after every pixel of the tile saturated contribute nothing
    for (uint32_t i = stop + lane; !ATOMIC && i < rg.y; i += 32) {
        const uint32_t j = pvals[i];
        const uint32_t p = pair_index(roffj, rec_[j].win, j, tx, ty);
        if ((uint64_t)p >= cap) continue;
#pragma unroll
        for (int q = 0; q < 9; ++q) partials[(uint64_t)p * 9 + q] = 0;
    }
    loss = warp_sum<double>(loss);
    if (lane == 0) tile_loss[tile] = loss;
#ifdef SS_BWD_STATS
    if (lane == 0)
        for (int k = 0; k < 6; ++k) atomicAdd(&g_bwd_stats[k], st[k]);
#endif
}

// ---------------------------------------------------------------- K5, float32 with paired rows
// The float32 forward walks a lane's 8 pixels as 4 row pairs (q = 2g, 2g + 1).
// The two pixels of a pair are independent chains of identical arithmetic,
// so they share one packed FFMA2 / FMUL2 / FADD2 (sm_100 paired fp32): the
// per-pixel arithmetic issues half the instructions, with per-component
// results identical to k_blend_fwd<float>.  (The backward keeps scalar rows:
// its packed form needs ~115 registers and loses more to occupancy than it
// saves in issue slots, measured.)
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float& comp(float2& v, int h) { return h ? v.y : v.x; }

#ifndef SS_FWD2_MINB
#define SS_FWD2_MINB 8
#endif
template <bool COUNT>  // COUNT: accumulate the evaluated (pixel, splat) pairs (timing runs only)
__global__ void __launch_bounds__(32 * WPB, SS_FWD2_MINB) k_blend_fwd2(const uint2* __restrict__ ranges,
                                                         const uint32_t* __restrict__ pvals,
                                                         const double2* __restrict__ mu,
                                                         const SplatRec<float>* __restrict__ rec, int W, int H,
                                                         int tiles_x, int n_tiles, double bg0, double bg1, double bg2,
                                                         float* __restrict__ img, float* __restrict__ Tout,
                                                         uint32_t* __restrict__ tile_stop,
                                                         unsigned long long* __restrict__ eval_count,
                                                         const uint32_t* __restrict__ order) {
    SS_PDL_WAIT();
    __shared__ Staged<float> sm[WPB][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = blockIdx.x * WPB + warp;
    if (slot >= n_tiles) return;
    const int tile = order ? (int)order[slot] : slot;
    const int X0 = (tile % tiles_x) * TILE, Y0 = (tile / tiles_x) * TILE;
    const int lx = lane & 15, ly0 = lane >> 4;
    const float pxc = lane_centre<float>(lx, X0), pyc = lane_centre<float>(ly0, Y0);
    unsigned alive = 0;
#pragma unroll
    for (int q = 0; q < PPT; ++q)
        if (X0 + lx < W && Y0 + ly0 + 2 * q < H) alive |= 1u << q;
    float2 T[PPT / 2], C0[PPT / 2], C1[PPT / 2], C2[PPT / 2];
#pragma unroll
    for (int g = 0; g < PPT / 2; ++g) T[g] = f2(1.f), C0[g] = f2(0.f), C1[g] = f2(0.f), C2[g] = f2(0.f);
    const uint2 rg = ranges[tile];
    int last = -1;
    uint32_t evals = 0;
    Staged<float>* my = sm[warp];
    const float2 cap = f2((float)ALPHA_CAP);
    for (uint32_t b0 = rg.x; b0 < rg.y; b0 += 32) {
        if (!__any_sync(0xffffffffu, alive)) break;
        const uint32_t i = b0 + lane;
        if (i < rg.y) {
            const uint32_t j = pvals[i];
            stage(my[lane], mu[j], rec[j], X0, Y0);
        }
        __syncwarp();
        const int nb = (int)min(32u, rg.y - b0);
        for (int k = 0; k < nb; ++k) {
            const Staged<float> s = my[k];
            const unsigned act = lane_mask(s, lx, ly0) & alive;
            if (!act) continue;
            last = (int)(b0 - rg.x) + k;
            if (COUNT) evals += __popc(act);
            PixelGeom<float, true> pg(s, pxc, pyc);
            const unsigned wact = __reduce_or_sync(__activemask(), act);
            const float2 cK = f2(pg.cK), Bx = f2(pg.Bx2), Ax = f2(pg.Ax2), o = f2(s.o);
#pragma unroll
            for (int g = 0; g < PPT / 2; ++g) {
                if (!((wact >> (2 * g)) & 3u)) continue;  // warp-uniform: no lane needs these rows
                const float2 y = add2(f2(pg.dy0), make_float2((float)(4 * g), (float)(4 * g + 2)));
                const float2 e = fma2(fma2(cK, y, Bx), y, Ax);
                float2 G;
                G.x = (act >> (2 * g)) & 1u ? ss_ex2(e.x) : 0.f;
                G.y = (act >> (2 * g + 1)) & 1u ? ss_ex2(e.y) : 0.f;
                float2 alpha = mul2(o, G);
                alpha.x = fminf(alpha.x, cap.x);
                alpha.y = fminf(alpha.y, cap.y);
                const float2 w = mul2(alpha, T[g]);
                C0[g] = fma2(w, f2(s.c0), C0[g]);
                C1[g] = fma2(w, f2(s.c1), C1[g]);
                C2[g] = fma2(w, f2(s.c2), C2[g]);
                T[g] = add2(T[g], neg2(w));
                gate_t(alive, T[g].x, 1u << (2 * g));
                gate_t(alive, T[g].y, 1u << (2 * g + 1));
            }
        }
        __syncwarp();
    }
    last = __reduce_max_sync(0xffffffffu, last + 1);
    if (lane == 0 && tile_stop) tile_stop[tile] = (uint32_t)last;
    if (COUNT) {
        evals = __reduce_add_sync(0xffffffffu, evals);
        if (lane == 0 && evals) atomicAdd(eval_count, (unsigned long long)evals);
    }
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
        const int px = X0 + lx, py = Y0 + ly0 + 2 * q;
        if (px < W && py < H) {
            const int64_t p = (int64_t)py * W + px;
            const float t = comp(T[q >> 1], q & 1);
            img[3 * p + 0] = comp(C0[q >> 1], q & 1) + t * (float)bg0;
            img[3 * p + 1] = comp(C1[q >> 1], q & 1) + t * (float)bg1;
            img[3 * p + 2] = comp(C2[q >> 1], q & 1) + t * (float)bg2;
            if (Tout) Tout[p] = t;
        }
    }
}

// ---------------------------------------------------------------- K6, float32 with paired rows
// The float32 backward walks a lane's 8 pixels as 4 row pairs (rows
// ly0 + 4g and ly0 + 4g + 2), the pair's two independent chains in one
// packed FFMA2 / FMUL2 / FADD2 each: per pixel the arithmetic of
// k_blend_bwd<float> (same operations in the same order per component, so
// T, R and every per-pixel term are bit-identical), with the 9 per-splat
// sums kept per row-pair component and folded before the warp reduction.
#ifndef SS_BWD2_MINB
#define SS_BWD2_MINB 8
#endif
__global__ void __launch_bounds__(32 * WPB_BWD, SS_BWD2_MINB) k_blend_bwd2(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ pvals, const double2* __restrict__ mu,
    const SplatRec<float>* __restrict__ rec_, const uint64_t* __restrict__ roffj, const uint32_t* __restrict__ tile_stop,
    int W, int H, int tiles_x, int n_tiles, const float* __restrict__ img, const float* __restrict__ gt, double npx3,
    float* __restrict__ partials, double* __restrict__ tile_loss, const uint32_t* __restrict__ order, uint64_t pair_cap) {
    SS_PDL_WAIT();
    __shared__ Staged<float> sm[WPB_BWD][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = blockIdx.x * WPB_BWD + warp;
    if (slot >= n_tiles) return;
    const int tile = order ? (int)order[slot] : slot;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int X0 = tx * TILE, Y0 = ty * TILE;
    const int lx = lane & 15, ly0 = lane >> 4;
    const float pxc = lane_centre<float>(lx, X0), pyc = lane_centre<float>(ly0, Y0);
    const uint2 rg = ranges[tile];
    const uint32_t stop = rg.x + (tile_stop ? min(tile_stop[tile], rg.y - rg.x) : (rg.y - rg.x));

    float2 T[PPT / 2], Rr[PPT / 2], g0[PPT / 2], g1[PPT / 2], g2[PPT / 2];
    unsigned alive = 0;
    double loss = 0.0;
    const float inv = (float)(1.0 / npx3);
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
        const int px = X0 + lx, py = Y0 + ly0 + 2 * q;
        float t = 1.f, r = 0.f, gg[3] = {0.f, 0.f, 0.f};
        if (px < W && py < H) {
            alive |= 1u << q;
            const int64_t p = (int64_t)py * W + px;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float v = img[3 * p + c];
                const float diff = v - gt[3 * p + c];
                loss += fabs((double)diff);
                const float sg = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
                gg[c] = sg * inv;  // dL/dC = sign(C - gt) / (H W 3)  (optim.py:124-125)
                r += gg[c] * v;
            }
        }
        comp(T[q >> 1], q & 1) = t;
        comp(Rr[q >> 1], q & 1) = r;
        comp(g0[q >> 1], q & 1) = gg[0];
        comp(g1[q >> 1], q & 1) = gg[1];
        comp(g2[q >> 1], q & 1) = gg[2];
    }
    Staged<float>* my = sm[warp];
    const float2 cap = f2((float)ALPHA_CAP), one = f2(1.f);
    for (uint32_t b0 = rg.x; b0 < stop; b0 += 32) {
        const uint32_t i = b0 + lane;
        if (i < stop) {
            const uint32_t j = pvals[i];
            const SplatRec<float> rec = rec_[j];
            stage(my[lane], mu[j], rec, X0, Y0);
            my[lane].p = (int)pair_index(roffj, rec.win, j, tx, ty);
        }
        __syncwarp();
        const int nb = (int)min(32u, stop - b0);
        for (int k = 0; k < nb; ++k) {
            const Staged<float> s = my[k];
            const unsigned act = lane_mask(s, lx, ly0) & alive;
            float2 acc[9];
#pragma unroll
            for (int e = 0; e < 9; ++e) acc[e] = f2(0.f);
            if (act) {
                PixelGeom<float, true> pg(s, pxc, pyc);
                const unsigned wact = __reduce_or_sync(__activemask(), act);
                const float2 cK = f2(pg.cK), Bx = f2(pg.Bx2), Ax = f2(pg.Ax2), o = f2(s.o);
                const float2 c0 = f2(s.c0), c1 = f2(s.c1), c2 = f2(s.c2), sb = f2(s.b), sc = f2(s.c);
                const float2 adx0 = f2(pg.adx0), bdx0 = f2(pg.bdx0);
#pragma unroll
                for (int g = 0; g < PPT / 2; ++g) {
                    if (!((wact >> (2 * g)) & 3u)) continue;  // warp-uniform skip of the row pair
                    const float2 y = add2(f2(pg.dy0), make_float2((float)(4 * g), (float)(4 * g + 2)));
                    const float2 ex = fma2(fma2(cK, y, Bx), y, Ax);
                    float2 G;
                    G.x = (act >> (2 * g)) & 1u ? ss_ex2(ex.x) : 0.f;
                    G.y = (act >> (2 * g + 1)) & 1u ? ss_ex2(ex.y) : 0.f;
                    const float2 oG = mul2(o, G);
                    const bool open_x = oG.x < cap.x, open_y = oG.y < cap.y;
                    const float2 alpha = make_float2(open_x ? oG.x : cap.x, open_y ? oG.y : cap.y);
                    const float2 w = mul2(alpha, T[g]);
                    const float2 gcol = fma2(g2[g], c2, fma2(g1[g], c1, mul2(g0[g], c0)));
                    acc[0] = fma2(g0[g], w, acc[0]);
                    acc[1] = fma2(g1[g], w, acc[1]);
                    acc[2] = fma2(g2[g], w, acc[2]);
                    // dL/dalpha = sum_c gC_c (col_c T - S_c / (1 - alpha)), S = C - prefix - contrib
                    const float2 rest = fma2(neg2(w), gcol, Rr[g]);
                    const float2 oma = add2(one, neg2(alpha));
                    const float2 rc = make_float2(ss_rcp<float>(oma.x), ss_rcp<float>(oma.y));
                    const float2 dal = fma2(T[g], gcol, neg2(mul2(rest, rc)));
                    Rr[g] = rest;
                    const float2 dalm = make_float2(open_x ? dal.x : 0.f, open_y ? dal.y : 0.f);  // capped: no gradient
                    const float2 dG = mul2(dalm, G);
                    const float2 gp = mul2(dalm, alpha);
                    const float2 adx = fma2(sb, y, adx0);
                    const float2 ady = fma2(sc, y, bdx0);
                    const float2 gpx = mul2(gp, adx), gpy = mul2(gp, ady);
                    acc[3] = add2(acc[3], dG);
                    acc[4] = add2(acc[4], gpx);
                    acc[5] = add2(acc[5], gpy);
                    acc[6] = fma2(gpx, adx, acc[6]);
                    acc[7] = fma2(gpx, ady, acc[7]);
                    acc[8] = fma2(gpy, ady, acc[8]);
                    T[g] = add2(T[g], neg2(w));
                    gate_t(alive, T[g].x, 1u << (2 * g));
                    gate_t(alive, T[g].y, 1u << (2 * g + 1));
                }
            }
            float* out = partials + (uint64_t)(uint32_t)s.p * 9;
            const bool fits = (uint64_t)(uint32_t)s.p < pair_cap;
            if (__any_sync(0xffffffffu, act != 0)) {
                float a8[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) a8[e] = acc[e].x + acc[e].y;
                const float y = warp_reduce8<float>(a8, lane);
                const float z = warp_sum<float>(acc[8].x + acc[8].y);
                if ((lane & 3) == 0 && fits) {
                    const int e = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
                    out[e] = e >= 6 ? 0.5f * y : y;
                }
                if (lane == 0 && fits) out[8] = 0.5f * z;
            } else if (lane < 9 && fits) {
                out[lane] = 0.f;
            }
        }
        __syncwarp();
    }
    // pairs after every pixel of the tile saturated contribute nothing
    for (uint32_t i = stop + lane; i < rg.y; i += 32) {
        const uint32_t j = pvals[i];
        const uint32_t p = pair_index(roffj, rec_[j].win, j, tx, ty);
        if ((uint64_t)p >= pair_cap) continue;
#pragma unroll
        for (int q = 0; q < 9; ++q) partials[(uint64_t)p * 9 + q] = 0.f;
    }
    loss = warp_sum<double>(loss);
    if (lane == 0) tile_loss[tile] = loss;
}

__global__ void k_loss_reduce(const double* __restrict__ tile_loss, int n, double inv_npx, double* __restrict__ out) {
    SS_PDL_WAIT();
    __shared__ double s[256];
    double t = 0;
    for (int i = threadIdx.x; i < n; i += 256) t += tile_loss[i];
    s[threadIdx.x] = t;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out += s[0] * inv_npx;
}

// ---------------------------------------------------------------- K7 chain rule
// (a) fixed-order sum of each splat's per-tile partials -> 9 values per input
//     row j.  Partials are stored in depth-rank order (a rank's pairs follow
//     its predecessor's), so a warp takes 32 consecutive ranks, stages their
//     contiguous partials through shared memory in chunks of whole pairs
//     (coalesced loads), and each lane sums its own rank's pairs in pair order.
#ifndef SP_PREFETCH
#define SP_PREFETCH 1
#endif
#ifndef SP_MINB
#define SP_MINB 4  // measured: 3 / 4 / 5 / 6 -> chain class 2.05 / 1.93 / 1.96 / 2.41 ms per step
#endif
template <typename R>
__global__ void __launch_bounds__(256, SP_MINB) k_sum_partials(const uint64_t* __restrict__ roff, const uint32_t* __restrict__ rcnt,
                                                      const uint32_t* __restrict__ dvals, const R* __restrict__ partials,
                                                      const SplatRec<R>* __restrict__ rec,
                                                      int64_t n_in, R* __restrict__ g9, uint64_t cap) {
    SS_PDL_WAIT();
    constexpr int PW = 4096 / (9 * sizeof(R));  // pairs per staged chunk (4 KB per warp)
    __shared__ R buf[8][PW * 9];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    R* sb = buf[warp];
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    for (int64_t r0 = ((int64_t)blockIdx.x * 8 + warp) * 32; r0 < n_in; r0 += nwarps * 32) {
        const int64_t r = r0 + lane;
        const bool valid = r < n_in;
        const uint64_t off = valid ? roff[r] : 0, cnt = valid ? rcnt[r] : 0;
        // the output row and its clamp mask first: their (random) loads
        // overlap the partial sums instead of following them
        const uint32_t j = valid ? dvals[r] : 0u;
        bool open[3] = {false, false, false};
        if (valid && cnt) {
#pragma unroll
            for (int c = 0; c < 3; ++c) open[c] = clamp_open(rec[j].col[c]);
        }
        const uint64_t P0 = __shfl_sync(0xffffffffu, off, 0);
        uint64_t end = valid ? off + cnt : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const uint64_t t = __shfl_xor_sync(0xffffffffu, end, o);
            end = t > end ? t : end;
        }
        end = end < cap ? end : cap;  // an overflowed call (flagged): never read past the partials
        R g[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // in the blend precision (fixed order: deterministic)
        for (uint64_t c0 = P0; c0 < end; c0 += PW) {
            const uint64_t c1 = min(c0 + PW, end);
            const int nf = (int)(c1 - c0) * 9;
            const R* src = partials + c0 * 9;
#if SP_PREFETCH
            if (c1 < end) {  // the next chunk into L1 while this one is summed
                const int nn = (int)(min(c1 + PW, end) - c1) * 9;
                for (int k = lane * (32 / (int)sizeof(R)); k < nn; k += 32 * (32 / (int)sizeof(R)))
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(partials + c1 * 9 + k));
            }
#endif
            for (int k = lane; k < nf; k += 32) sb[k] = src[k];
            __syncwarp();
            const uint64_t a = off > c0 ? off : c0, b = off + cnt < c1 ? off + cnt : c1;
            for (uint64_t p = a; p < b; ++p) {
                const R* q = sb + (p - c0) * 9;
#pragma unroll
                for (int e = 0; e < 9; ++e) g[e] += q[e];
            }
            __syncwarp();
        }
        if (valid) {
            SS_ASSERT(j < (uint64_t)n_in);
            R* o = g9 + (int64_t)j * 9;
            if (cnt) {  // dL/dcolour through the clamp: zero where the forward clamped (optim.py:176-177)
#pragma unroll
                for (int c = 0; c < 3; ++c) g[c] = open[c] ? g[c] : (R)0;
            }
#pragma unroll
            for (int e = 0; e < 9; ++e) o[e] = g[e];
        }
    }
}

// (b) the chain rule in row order
#ifndef CHAIN_FAST_NORM
#define CHAIN_FAST_NORM 1  // fp32 chain rule: norms and their inverses from one rsqrt
#endif
#ifndef CHAIN_FAST_EXP
#define CHAIN_FAST_EXP 1  // fp32 chain rule: the hardware exp2-based __expf (tolerance-checked)
#endif
template <typename T> __device__ __forceinline__ T t_exp(T x);
template <> __device__ __forceinline__ float t_exp<float>(float x) { return CHAIN_FAST_EXP ? __expf(x) : expf(x); }
template <> __device__ __forceinline__ double t_exp<double>(double x) { return exp(x); }

// a / b in the chain rule: fp32 multiplies by the reciprocal ib = 1 / b (one
// division per divisor instead of one per quotient; the fp32 chain rule is
// tolerance-checked against the reference), fp64 divides exactly
// |v| and 1 / |v| from v.v: fp32 from one rsqrt (x * rsqrt(x) for the norm),
// fp64 the IEEE sqrt and its reciprocal
template <typename T>
__device__ __forceinline__ void norm_and_inverse(T x, T& n, T& inv) {
    if constexpr (sizeof(T) == 4) {
        if (CHAIN_FAST_NORM) {
            inv = rsqrtf(x);
            n = x * inv;
            return;
        }
    }
    n = sqrt(x);
    inv = (T)1 / n;
}

template <typename T>
__device__ __forceinline__ T cdiv(T a, T b, T ib) {
    if constexpr (sizeof(T) == 4) return a * ib;
    else return a / b;
}

// The chain rule of one (row, view) (ref optim.py:170-268): adds the row's
// parameter gradients of this view into acc (means 3, log scales 3,
// quaternion 4, opacity 1) with the same fp32 additions the gradient buffer
// would see, and writes the row's SH record for k_sh_grad.
template <typename T, int DEG, typename PT = float>
__device__ __forceinline__ void chain_row(const ss_model& m, const ss_camera& cam, const ss_light& L, int64_t row,
                                          const T* g, float* acc, float4* __restrict__ shrec_row) {
    constexpr int B = ss_sh_bases(DEG);
    const ParamView<PT> pv(m);
    T Rc[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) Rc[i][k] = (T)cam.rot_cw[3 * i + k];
    const T fx = (T)cam.fx, fy = (T)cam.fy;
    const T ldir[3] = {(T)L.direction[0], (T)L.direction[1], (T)L.direction[2]};
    // ---- appearance first (the SH registers die early)
    T d[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) d[i] = (T)((double)pv.means[row * 3 + i] - cam.position[i]);
    T dist, idist;
    norm_and_inverse(d[0] * d[0] + d[1] * d[1] + d[2] * d[2], dist, idist);
    const T vdir[3] = {cdiv(d[0], dist, idist), cdiv(d[1], dist, idist), cdiv(d[2], dist, idist)};
    const PT* lsp = pv.ls + row * 3;
    int axis;
    {
        const double l0 = lsp[0], l1 = lsp[1], l2 = lsp[2];
        const double mn = fmin(l0, fmin(l1, l2)) + SS_AXIS_MARGIN;
        axis = (l0 <= mn) ? 0 : ((l1 <= mn) ? 1 : 2);
    }
    T u[4];
    T qn, iqn;
    {
        const PT* qp = pv.quats + row * 4;
        const T q0 = qp[0], q1 = qp[1], q2 = qp[2], q3 = qp[3];
        norm_and_inverse(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3, qn, iqn);
        u[0] = cdiv(q0, qn, iqn); u[1] = cdiv(q1, qn, iqn); u[2] = cdiv(q2, qn, iqn); u[3] = cdiv(q3, qn, iqn);
    }
    const T w = u[0], qx = u[1], qy = u[2], qz = u[3];
    T Rq[3][3];
    Rq[0][0] = 1 - 2 * (qy * qy + qz * qz); Rq[0][1] = 2 * (qx * qy - w * qz); Rq[0][2] = 2 * (qx * qz + w * qy);
    Rq[1][0] = 2 * (qx * qy + w * qz); Rq[1][1] = 1 - 2 * (qx * qx + qz * qz); Rq[1][2] = 2 * (qy * qz - w * qx);
    Rq[2][0] = 2 * (qx * qz - w * qy); Rq[2][1] = 2 * (qy * qz + w * qx); Rq[2][2] = 1 - 2 * (qx * qx + qy * qy);
    // dL/dcolour arrives masked by the forward's clamp (the partial sums zero
    // the channels whose pre-clamp colour was outside (0, 1): optim.py:176-177
    // with the preprocess's own color_pre, as the reference reads
    // prepared.color_pre), so the shading is not re-evaluated here; only its
    // terms the gradient needs: the normal proxy's cosine, visibility, albedo
    // (ss_shade_v's expressions) and, for the view-direction path, the SH dot.
    T gc[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) gc[c] = g[c];
    T gv[3] = {0, 0, 0};
    T albedo[3];
    T cosv, vis, sgn_s;
    {
        T nhat[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) nhat[i] = axis == 0 ? Rq[i][0] : (axis == 1 ? Rq[i][1] : Rq[i][2]);
        sgn_s = nhat[0] * (T)-L.direction[0] + nhat[1] * (T)-L.direction[1] + nhat[2] * (T)-L.direction[2];
        cosv = fabs(sgn_s);
        vis = (T)pv.vis[row];
        const PT* shr = pv.sh + row * 3 * B;
#pragma unroll
        for (int c = 0; c < 3; ++c) albedo[c] = (T)SS_SH_C0 * (T)shr[c * B] + (T)0.5;
        if constexpr (DEG > 0) {
            if (gc[0] != (T)0 || gc[1] != (T)0 || gc[2] != (T)0) {
                PT sh[3 * B];
                ss_load_sh<DEG, PT>(shr, sh);
                T coef[B];
#pragma unroll
                for (int k = 0; k < B; ++k) coef[k] = sh[k] * gc[0] + sh[B + k] * gc[1] + sh[2 * B + k] * gc[2];
                ss_sh_grad_dot<DEG, T>(vdir, coef, gv);
            }
        }
    }
    // SH coefficient gradients: written by k_sh_grad from this compact record
    shrec_row[0] = make_float4((float)gc[0], (float)gc[1], (float)gc[2], (float)(cosv * vis));
    shrec_row[1] = make_float4((float)vdir[0], (float)vdir[1], (float)vdir[2], 1.0f);

    // ---- geometry: mu_cam, J, Sigma3d, cov (render.py:246-267)
    T mc[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) mc[k] = d[0] * Rc[0][k] + d[1] * Rc[1][k] + d[2] * Rc[2][k];
    const T x = mc[0], y = mc[1], z = mc[2];
    const T iz = (T)1 / z, z2 = z * z;
    const T iz2 = (T)1 / z2;  // (fp32: the quotients below multiply by it; fp64 divides)
    const T J00 = fx * iz, J02 = cdiv(-fx * x, z2, iz2), J11 = fy * iz, J12 = cdiv(-fy * y, z2, iz2);
    T S2[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) S2[k] = t_exp<T>((T)2 * (T)lsp[k]);
    T S3[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = i; k < 3; ++k) {
            S3[i][k] = Rq[i][0] * S2[0] * Rq[k][0] + Rq[i][1] * S2[1] * Rq[k][1] + Rq[i][2] * S2[2] * Rq[k][2];
            S3[k][i] = S3[i][k];
        }
    T tm[3][3], cov[3][3];  // cov = W S3 W^T, W[i][k] = Rc[k][i]
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int l = 0; l < 3; ++l) tm[i][l] = Rc[0][i] * S3[0][l] + Rc[1][i] * S3[1][l] + Rc[2][i] * S3[2][l];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = i; k < 3; ++k) {
            cov[i][k] = tm[i][0] * Rc[0][k] + tm[i][1] * Rc[1][k] + tm[i][2] * Rc[2][k];
            cov[k][i] = cov[i][k];
        }
    // ---- optim.py:180-195
    const T g00 = g[6], g01 = g[7], g11 = g[8];
    T JC0[3], JC1[3];
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        JC0[l] = J00 * cov[0][l] + J02 * cov[2][l];
        JC1[l] = J11 * cov[1][l] + J12 * cov[2][l];
    }
    T gJ0[3], gJ1[3];
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        gJ0[l] = 2 * (g00 * JC0[l] + g01 * JC1[l]);
        gJ1[l] = 2 * (g01 * JC0[l] + g11 * JC1[l]);
    }
    // gV = J^T G2 J (J rows: [J00, 0, J02], [0, J11, J12])
    const T Jr0[3] = {J00, 0, J02}, Jr1[3] = {0, J11, J12};
    T JG0[3], JG1[3];
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        JG0[l] = g00 * Jr0[l] + g01 * Jr1[l];
        JG1[l] = g01 * Jr0[l] + g11 * Jr1[l];
    }
    T gV[3][3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int l = 0; l < 3; ++l) gV[k][l] = Jr0[k] * JG0[l] + Jr1[k] * JG1[l];
    T G3[3][3];  // R_cw gV R_cw^T
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int l = 0; l < 3; ++l) tm[i][l] = Rc[i][0] * gV[0][l] + Rc[i][1] * gV[1][l] + Rc[i][2] * gV[2][l];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) G3[i][k] = tm[i][0] * Rc[k][0] + tm[i][1] * Rc[k][1] + tm[i][2] * Rc[k][2];
    const T gm0 = g[4], gm1 = g[5];
    const T z3 = z2 * z;
    const T iz3 = (T)1 / z3;
    const T fxz2 = cdiv(-fx, z2, iz2), fyz2 = cdiv(-fy, z2, iz2);
    T gmc[3];
    gmc[0] = J00 * gm0 + gJ0[2] * fxz2;
    gmc[1] = J11 * gm1 + gJ1[2] * fyz2;
    gmc[2] = J02 * gm0 + J12 * gm1 + gJ0[0] * fxz2 + gJ1[1] * fyz2 + gJ0[2] * cdiv(2 * fx * x, z3, iz3) +
             gJ1[2] * cdiv(2 * fy * y, z3, iz3);
    T gmean[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) gmean[i] = Rc[i][0] * gmc[0] + Rc[i][1] * gmc[1] + Rc[i][2] * gmc[2];
    if constexpr (DEG > 0) {  // view-direction path (optim.py:235-240)
        const T vg = vdir[0] * gv[0] + vdir[1] * gv[1] + vdir[2] * gv[2];
#pragma unroll
        for (int i = 0; i < 3; ++i) gmean[i] += cdiv(gv[i] - vdir[i] * vg, dist, idist);
    }
    // ---- scales and rotation (optim.py:204-218)
    T gls[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        T t = 0;
#pragma unroll
        for (int b2 = 0; b2 < 3; ++b2)
#pragma unroll
            for (int c = 0; c < 3; ++c) t += Rq[b2][k] * G3[b2][c] * Rq[c][k];
        gls[k] = t * 2 * S2[k];
    }
    T gR[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            T t = 0;
#pragma unroll
            for (int b2 = 0; b2 < 3; ++b2) t += (G3[i][b2] + G3[b2][i]) * Rq[b2][c];
            gR[i][c] = t * S2[c];
        }
    T gcos = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) gcos += gc[c] * (albedo[c] * (T)L.intensity[c]);
    gcos *= vis;
    const T gs = gcos * (sgn_s > 0 ? (T)1 : (sgn_s < 0 ? (T)-1 : (T)0));
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (k == axis) gR[i][k] += gs * -ldir[i];
    // quaternion through R(u), u = q / |q| (optim.py:87-110)
    const T dR[4][3][3] = {
        {{0, -2 * qz, 2 * qy}, {2 * qz, 0, -2 * qx}, {-2 * qy, 2 * qx, 0}},
        {{0, 2 * qy, 2 * qz}, {2 * qy, -4 * qx, -2 * w}, {2 * qz, 2 * w, -4 * qx}},
        {{-4 * qy, 2 * qx, 2 * w}, {2 * qx, 0, 2 * qz}, {-2 * w, 2 * qz, -4 * qy}},
        {{-4 * qz, -2 * w, 2 * qx}, {2 * w, -4 * qz, 2 * qy}, {2 * qx, 2 * qy, 0}}};
    T h[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        T t = 0;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int jj = 0; jj < 3; ++jj) t += gR[i][jj] * dR[c][i][jj];
        h[c] = t;
    }
    const T udh = u[0] * h[0] + u[1] * h[1] + u[2] * h[2] + u[3] * h[3];
    const T op = (T)1 / ((T)1 + t_exp<T>(-(T)pv.logit[row]));
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        acc[i] += (float)gmean[i];
        acc[3 + i] += (float)gls[i];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[6 + k] += (float)cdiv(h[k] - u[k] * udh, qn, iqn);
    acc[10] += (float)(g[3] * op * (1 - op));
}

// gradient layout offsets of a row's 11 non-SH entries (see ss_grad_layout;
// `a` is the layout's row count -- the active count, or a row shard's length
// in the view-sharded step -- and `row` is relative to the layout's first row)
__device__ __forceinline__ void grad_row_load(const float* grad, int64_t a, int64_t row, float* acc) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        acc[i] = grad[row * 3 + i];
        acc[3 + i] = grad[3 * a + row * 3 + i];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[6 + k] = grad[6 * a + row * 4 + k];
    acc[10] = grad[10 * a + row];
}
__device__ __forceinline__ void grad_row_store(float* grad, int64_t a, int64_t row, const float* acc) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        grad[row * 3 + i] = acc[i];
        grad[3 * a + row * 3 + i] = acc[3 + i];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) grad[6 * a + row * 4 + k] = acc[6 + k];
    grad[10 * a + row] = acc[10];
}

// Chain rule in the blend precision T (fp32 for the throughput path, fp64
// for the parity path); the normal-proxy axis pick repeats the preprocess's
// fp64 comparison so both passes agree on it.
template <typename T, int DEG, typename PT = float>
__global__ void __launch_bounds__(128, 4) k_chain(ss_model m, ss_camera cam, ss_light L, const int64_t* __restrict__ subset,
                        const uint32_t* __restrict__ rinv, const T* __restrict__ g9, int64_t n_in, int cutoff,
                        float* __restrict__ grad, float4* __restrict__ shrec) {
    SS_PDL_WAIT();
    const int64_t a = m.active_count;
    // row order: parameter reads and gradient writes are coalesced
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_in; j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t r = rinv[j];
        if (r == ~0u) continue;
        const int64_t row = subset ? subset[j] : j;
        if (row >= a) continue;
        T g[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) g[e] = g9[j * 9 + e];
        float acc[11];
        grad_row_load(grad, a, row, acc);
        chain_row<T, DEG, PT>(m, cam, L, row, g, acc, shrec + row * 2);
        grad_row_store(grad, a, row, acc);
    }
}

// The step's views in one pass (ss_chain_views): per row, every view in
// order, the gradient read and written once.
constexpr int CV_MAX_VIEWS = 16;
struct ChainViews {
    ss_camera cam[CV_MAX_VIEWS];
    ss_light light[CV_MAX_VIEWS];
    const float* g9[CV_MAX_VIEWS];
    const uint32_t* rinv[CV_MAX_VIEWS];
};

#ifndef CV_MINB
#define CV_MINB 4  // measured (chain class per step, with the clamp mask from the partial sums): 2 / 3 / 4 -> 2.09 / 2.09 / 1.97 ms
#endif
#ifndef CV_PREFETCH
#define CV_PREFETCH 1
#endif
// Inputs j in [j0, j1) (row = subset[j], or j); the gradient layout starts at
// row0 with ld rows per group (ld = a, row0 = 0 on one GPU; a row shard in
// the view-sharded step, whose g9 / rinv pointers are offset to be indexed by j).
// SH coefficient gradients of one row from its per-view records (gc, cos vis,
// view dir): g_sh[c, b] += gc_{v,c} K_{v,c,b} in view order with
//   K = [b < BL] ambient[c][b] + [b >= 1] Y_b(view dir) + [b == 0] C0 I_c cos vis
// (ambient light; without it K = Y_b + [b == 0] C0 I_c cos vis) -- ref
// optim.py:221-233: the ambient product, the view-dependent basis and the
// direct-light term through albedo_est = C0 dc + 0.5.  `rec` is the row's
// record of view v at rec[v * stride]; io holds the row's 3B entries.
// per view, the SH-gradient constants in float (ss_light's doubles converted
// once per block instead of once per row): amb[v][c][b] = [b < BL]
// ambient[c][b] (zero without ambient light), dc[v][c] = C0 I_c, has_amb[v]
struct ShConst {
    float amb[CV_MAX_VIEWS][3][16];
    float dc[CV_MAX_VIEWS][3];
    int has_amb[CV_MAX_VIEWS];
};

template <int DEG>
__device__ __forceinline__ void sh_const_load(const ChainViews* V, int nv, ShConst& K) {
    constexpr int B = ss_sh_bases(DEG);
    for (int i = threadIdx.x; i < nv * 3 * B; i += blockDim.x) {
        const int v = i / (3 * B), r = i - v * 3 * B, c = r / B, b = r - c * B;
        const ss_light& L = V->light[v];
        const int BL = L.ambient_bands < B ? L.ambient_bands : B;
        K.amb[v][c][b] = b < BL ? (float)L.ambient[c * L.ambient_bands + b] : 0.f;
        if (b == 0) K.dc[v][c] = (float)(SS_SH_C0 * L.intensity[c]);
        if (r == 0) K.has_amb[v] = L.ambient_bands != 0;
    }
}

// SH coefficient gradients of one row from its per-view records (gc, cos vis,
// view dir): g_sh[c, b] += gc_{v,c} K_{v,c,b} in view order with
//   K = [b < BL] ambient[c][b] + [b >= 1] Y_b(view dir) + [b == 0] C0 I_c cos vis
// (ambient light; without it K = Y_b + [b == 0] C0 I_c cos vis) -- ref
// optim.py:221-233: the ambient product, the view-dependent basis and the
// direct-light term through albedo_est = C0 dc + 0.5.  `rec` is the row's
// record of view v at rec[v * stride]; io holds the row's 3B entries.  The
// views' first record halves are loaded up front (their loads overlap).
template <int DEG>
__device__ __forceinline__ void sh_grad_row(const ShConst& K, int nv, const float4* rec, int stride, float* io) {
    constexpr int B = ss_sh_bases(DEG);
    float4 r0s[CV_MAX_VIEWS];
#pragma unroll
    for (int v = 0; v < CV_MAX_VIEWS; ++v)
        if (v < nv) r0s[v] = rec[(size_t)v * stride];
    float acc[3 * B];
    bool loaded = false;
#pragma unroll
    for (int v = 0; v < CV_MAX_VIEWS; ++v) {
        if (v >= nv) break;
        const float4 r0 = r0s[v];
        if (r0.x == 0.f && r0.y == 0.f && r0.z == 0.f) continue;  // clamped colour or not visible
        if (!loaded) {
#pragma unroll
            for (int e = 0; e < 3 * B; ++e) acc[e] = io[e];
            loaded = true;
        }
        const float4 r1 = rec[(size_t)v * stride + 1];
        const float dir[3] = {r1.x, r1.y, r1.z};
        float Y[B];
        ss_sh_eval<DEG, float>(dir, Y);
        const bool amb = K.has_amb[v];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float gcc = c == 0 ? r0.x : (c == 1 ? r0.y : r0.z);
            if (gcc == 0.f) continue;
#pragma unroll
            for (int b = 0; b < B; ++b) {
                float kv;
                if (!amb) kv = Y[b];
                else kv = K.amb[v][c][b] + (b >= 1 ? Y[b] : 0.f);
                if (b == 0) kv += K.dc[v][c] * r0.w;
                acc[c * B + b] = fmaf(gcc, kv, acc[c * B + b]);
            }
        }
    }
    if (loaded) {
#pragma unroll
        for (int e = 0; e < 3 * B; ++e) io[e] = acc[e];
    }
}

constexpr int CVB = 128;  // rows (threads) per block of k_chain_views / k_sh_grad_rows
__host__ __device__ constexpr int cv_sh_stride(int B) { return (3 * B + 1) | 1; }  // odd: conflict-free rows

// Inputs j in [j0, j1) (row = subset[j], or j); the gradient layout starts at
// row0 with ld rows per group (ld = a, row0 = 0 on one GPU; a row shard in
// the view-sharded step, whose g9 / rinv pointers are offset to be indexed
// by j).  Per row every view in order, the 11 non-SH gradient entries read
// and written once; each (view, row) leaves its compact SH record in shrec
// for k_sh_grad_rows.
template <int DEG>
__global__ void __launch_bounds__(CVB, CV_MINB) k_chain_views(ss_model m, const __grid_constant__ ChainViews Vp, int nv,
                                                        const int64_t* __restrict__ subset, int64_t j0, int64_t j1,
                                                        int64_t row0, int64_t ld,
                                                        float* __restrict__ grad, float4* __restrict__ shrec, int init) {
    SS_PDL_WAIT();
    const ChainViews* V = &Vp;  // the views ride in the kernel parameters (no host-to-device copy)
    const int64_t a = m.active_count;
    for (int64_t j = j0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < j1; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = subset ? subset[j] : j;
        if (row >= a) continue;
        const int64_t rel = row - row0;
        float acc[11];
        bool any = init != 0;  // init: the layout was not cleared -- start from zero, always store
        if (init) {
#pragma unroll
            for (int e = 0; e < 11; ++e) acc[e] = 0.f;
        }
#if CV_PREFETCH
        // the next views' screen-space gradients into L1 while this view's chain runs
        for (int v = 1; v < nv; ++v) asm volatile("prefetch.global.L1 [%0];" ::"l"(V->g9[v] + j * 9));
#endif
        // the row's visibility in every view first (independent loads, one mask)
        unsigned vis = 0;
#pragma unroll
        for (int v = 0; v < CV_MAX_VIEWS; ++v)
            if (v < nv && V->rinv[v][j] != ~0u) vis |= 1u << v;
        for (int v = 0; v < nv; ++v) {
            if (!((vis >> v) & 1u)) {  // not visible: a zero record
                shrec[((int64_t)v * ld + rel) * 2] = make_float4(0.f, 0.f, 0.f, 0.f);
                continue;
            }
            if (!any) {
                grad_row_load(grad, ld, rel, acc);
                any = true;
            }
            float g[9];
#pragma unroll
            for (int e = 0; e < 9; ++e) g[e] = V->g9[v][j * 9 + e];
            chain_row<float, DEG>(m, V->cam[v], V->light[v], row, g, acc, shrec + ((int64_t)v * ld + rel) * 2);
        }
        if (any) grad_row_store(grad, ld, rel, acc);
    }
}

// The SH gradients of rows [0, rows) of the layout from the step's records
// (sh_grad_row), one thread per row; a block's SH rows are contiguous, so
// they are staged through shared memory (coalesced reads and writes, the
// row's 3B entries in registers across the views).
#ifndef SHR_MINB
#define SHR_MINB 3  // measured (chain class per step, views' first records loaded up front): 2 / 3 / 4 / 5 / 6 -> 1.770 / 1.773 / 1.836 / 2.390 / 2.696 ms
#endif
template <int DEG>
__global__ void __launch_bounds__(CVB, SHR_MINB) k_sh_grad_rows(const __grid_constant__ ChainViews Vp, int nv,
                                                      const float4* __restrict__ shrec, int64_t rows, int64_t ld,
                                                      float* __restrict__ grad_sh, int init) {
    SS_PDL_WAIT();
    constexpr int B = ss_sh_bases(DEG);
    constexpr int S = cv_sh_stride(B);
    __shared__ float s_sh[CVB * S];
    __shared__ ShConst K;
    sh_const_load<DEG>(&Vp, nv, K);
    const int t = threadIdx.x;
    for (int64_t rb = (int64_t)blockIdx.x * CVB; rb < rows; rb += (int64_t)gridDim.x * CVB) {
        const int nr = (int)min((int64_t)CVB, rows - rb);
        float* gb = grad_sh + rb * 3 * B;
        // init: the layout was not cleared -- the rows start from zero
        for (int e = t; e < nr * 3 * B; e += CVB) s_sh[(e / (3 * B)) * S + e % (3 * B)] = init ? 0.f : gb[e];
        __syncthreads();
        if (t < nr) sh_grad_row<DEG>(K, nv, shrec + (rb + t) * 2, (int)(2 * ld), s_sh + t * S);
        __syncthreads();
        for (int e = t; e < nr * 3 * B; e += CVB) gb[e] = s_sh[(e / (3 * B)) * S + e % (3 * B)];
        __syncthreads();
    }
}

// SH coefficient gradients, one thread per (row, channel, basis) entry
// (ref optim.py:221-233): ambient product, view-dependent basis and the
// direct-light term through albedo_est = C0 dc + 0.5.
constexpr int SHG_ROWS = 64;  // rows per block in k_sh_grad

template <int DEG>
__global__ void __launch_bounds__(256) k_sh_grad(ss_light L, const float4* __restrict__ shrec, int64_t a,
                                                 float* __restrict__ grad_sh) {
    SS_PDL_WAIT();
    constexpr int B = ss_sh_bases(DEG);
    __shared__ float s_y[SHG_ROWS][B + 1];
    __shared__ float4 s_r0[SHG_ROWS];
    const int64_t row0 = (int64_t)blockIdx.x * SHG_ROWS;
    const int nrows = (int)min((int64_t)SHG_ROWS, a - row0);
    if (threadIdx.x < nrows) {  // one thread per row: the basis values once
        const float4 r0 = shrec[2 * (row0 + threadIdx.x)];
        const float4 r1 = shrec[2 * (row0 + threadIdx.x) + 1];
        const float v[3] = {r1.x, r1.y, r1.z};
        float Y[B];
        ss_sh_eval<DEG, float>(v, Y);
#pragma unroll
        for (int k = 0; k < B; ++k) s_y[threadIdx.x][k] = Y[k];
        s_r0[threadIdx.x] = r0;
    }
    __syncthreads();
    const int BL = L.ambient_bands < B ? L.ambient_bands : B;
    const int n = nrows * 3 * B;
    float* out = grad_sh + row0 * 3 * B;
    if constexpr (B % 4 == 0) {  // float4 per thread: 4 bases of one (row, channel)
        if ((reinterpret_cast<uintptr_t>(out) & 15) == 0) {
            for (int e4 = threadIdx.x; e4 < n / 4; e4 += blockDim.x) {
                const int e = 4 * e4;
                const int r = e / (3 * B), rem = e - r * 3 * B, c = rem / B, b0 = rem - c * B;
                const float4 r0 = s_r0[r];
                const float gcc = c == 0 ? r0.x : (c == 1 ? r0.y : r0.z);
                if (gcc == 0.f) continue;
                float v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int b = b0 + k;
                    const float yb = s_y[r][b];
                    if (L.ambient_bands == 0) {
                        v[k] = gcc * yb;
                    } else {
                        v[k] = (b < BL ? gcc * (float)L.ambient[c * L.ambient_bands + b] : 0.f) + (b >= 1 ? gcc * yb : 0.f);
                    }
                }
                if (b0 == 0) v[0] += gcc * (float)(SS_SH_C0 * L.intensity[c]) * r0.w;
                float4* o4 = reinterpret_cast<float4*>(out + e);
                float4 cur = *o4;
                cur.x += v[0]; cur.y += v[1]; cur.z += v[2]; cur.w += v[3];
                *o4 = cur;
            }
            return;
        }
    }
    for (int e = threadIdx.x; e < n; e += blockDim.x) {  // coalesced over the block's contiguous rows
        const int r = e / (3 * B), rem = e - r * 3 * B, c = rem / B, b = rem - c * B;
        const float4 r0 = s_r0[r];
        const float gcc = c == 0 ? r0.x : (c == 1 ? r0.y : r0.z);
        if (gcc == 0.f) continue;  // clamped colour or row not visible in this view
        const float yb = s_y[r][b];
        float v;
        if (L.ambient_bands == 0) {
            v = gcc * yb;
        } else {
            v = (b < BL ? gcc * (float)L.ambient[c * L.ambient_bands + b] : 0.f) + (b >= 1 ? gcc * yb : 0.f);
        }
        if (b == 0) v += gcc * (float)(SS_SH_C0 * L.intensity[c]) * r0.w;
        out[e] += v;
    }
}

// ---------------------------------------------------------------- tile order
// Tiles are walked longest-first (work = list length, or the forward's stop
// index for the backward): the blocks holding the longest walks start in the
// first wave instead of forming the tail, and tiles of similar length share a
// block (a block retires with its slowest tile).  Counting sort on the work,
// one block; ties in any order (every tile's results are independent of the
// schedule).
constexpr int ORDER_BUCKETS = 4096;

__global__ void __launch_bounds__(1024) k_tile_order(const uint2* __restrict__ ranges,
                                                     const uint32_t* __restrict__ stop, int n_tiles,
                                                     uint32_t* __restrict__ order) {
    SS_PDL_WAIT();
    __shared__ uint32_t h[ORDER_BUCKETS];
    __shared__ uint32_t ws[32];
    for (int i = threadIdx.x; i < ORDER_BUCKETS; i += blockDim.x) h[i] = 0;
    __syncthreads();
    auto bucket = [&](int t) {
        const uint2 r = ranges[t];
        uint32_t w = r.y - r.x;
        if (stop) w = min(w, stop[t]);
        return ORDER_BUCKETS - 1 - (int)min(w, (uint32_t)(ORDER_BUCKETS - 1));  // descending work
    };
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) atomicAdd(&h[bucket(t)], 1u);
    __syncthreads();
    // exclusive scan of the 4096 buckets: 4 per thread
    constexpr int PER = ORDER_BUCKETS / 1024;
    uint32_t v[PER], sum = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        v[k] = h[threadIdx.x * PER + k];
        sum += v[k];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
    }
    if (lane == 31) ws[warp] = incl;
    __syncthreads();
    uint32_t pre = 0;
    for (int w = 0; w < warp; ++w) pre += ws[w];
    uint32_t run = pre + incl - sum;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        h[threadIdx.x * PER + k] = run;
        run += v[k];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) order[atomicAdd(&h[bucket(t)], 1u)] = (uint32_t)t;
}

// ---------------------------------------------------------------- host
inline int gridn(ss_ctx* ctx, int64_t n, int block = 256) {
    int64_t g = (n + block - 1) / block;
#ifndef SS_GRID_CAP
#define SS_GRID_CAP 32
#endif
    int64_t cap = (int64_t)ctx->num_sms * SS_GRID_CAP;
    if (g > cap) g = cap;
    return g < 1 ? 1 : (int)g;
}

int validate(ss_ctx* ctx, const ss_model* m, const ss_camera* cam, const ss_render_opts* o) {
    if (!m || !cam || !o) return ss_fail(ctx, SS_ERR_INVALID, "null argument");
    if (m->sh_degree < 0 || m->sh_degree > 3) return ss_fail(ctx, SS_ERR_INVALID, "sh_degree must be 0..3");
    if (cam->width <= 0 || cam->height <= 0) return ss_fail(ctx, SS_ERR_INVALID, "bad image size");
    if (o->precision != 0 && o->precision != 1) return ss_fail(ctx, SS_ERR_INVALID, "precision must be 0 or 1");
    if (m->count < 0 || m->active_count < 0 || m->active_count > m->count)
        return ss_fail(ctx, SS_ERR_INVALID, "bad row counts");
    if (m->param_dtype != 0 && (m->param_dtype != 1 || o->precision != 1))
        return ss_fail(ctx, SS_ERR_INVALID, "float64 parameters need the fp64 blend (precision 1)");
    return SS_OK;
}

// The pair count of a binning on the device: n_pairs = min(total, cap); a
// call whose pairs exceed the capacity counts an overflow in status[0]
// (sticky: the optimizer step's Adam leaves the model alone while it is set)
// and every call raises status[1] to its pair count (the host's next capacity).
__global__ void k_clamp_pairs(const uint64_t* __restrict__ total, uint64_t cap, uint64_t* __restrict__ n_pairs,
                              int64_t* __restrict__ status) {
    SS_PDL_WAIT();
    const uint64_t t = *total;
    *n_pairs = t < cap ? t : cap;
    if (status) {
        if (t > cap) atomicAdd((unsigned long long*)&status[0], 1ull);
        atomicMax((unsigned long long*)&status[1], (unsigned long long)t);
    }
}

// K1..K4: preprocess, depth sort, count/scan/emit, tile sort, ranges.
// (tile, splat) pairs of a depth-ordered splat set: counts per rank, scan,
// warp-cooperative emission, stable tile sort, per-tile ranges.  Needs b's
// dkey64 (~0 = culled), dvals (input index by rank), rec and the geometry.
//
// Pair buffers are sized on the host.  With a status buffer and a known
// capacity (ctx->pair_cap) nothing is read back: the kernels take the pair
// count from the device and never touch more than the capacity (an overflow
// is flagged in status, see k_clamp_pairs).  Otherwise (no status, or the
// first call of a context) the count is read back once and sets the
// capacity for the calls that follow (1.1x + 64k pairs of headroom; a later
// overflow grows it through the caller, see optim.step).
template <typename R>
int bin_pairs(ss_ctx* ctx, Bins& b, int64_t* status) {
    cudaStream_t s = ctx->stream;
    const int64_t n = b.n_in;
    uint64_t* total = SS_SCRATCH(ctx, uint64_t, 1);
    b.n_pairs = SS_SCRATCH(ctx, uint64_t, 1);
    if (!total || !b.n_pairs) return SS_ERR_CUDA;
    ss_tic(ctx, KC_BIN);
    if (n > 0) {
        SS_CUDA(ctx, ss_launch((k_count<R>), dim3(gridn(ctx, n)), dim3(256), 0, s, b.dkey64, b.dvals, (const SplatRec<R>*)b.rec, n, b.rcnt, b.rinv));
        SS_CHECK_LAUNCH(ctx);
    }
    SS_TRY(ss_scan_u32_to_u64(ctx, b.rcnt, b.roff, n, total));
    ss_toc(ctx, KC_BIN);
    uint64_t cap;
#ifdef SS_FORCE_SYNC_BINS  // A/B measurements only: read every pair count back
    if (false) {
#else
    if (status && ctx->pair_cap > 0) {
#endif
        cap = (uint64_t)ctx->pair_cap;
    } else {
        SS_TRY(ss_read_u64(ctx, total, &cap));
        if (status) {
            const int64_t want = (int64_t)(cap + cap / 10 + 65536);
            if (want > ctx->pair_cap) ctx->pair_cap = want;
        }
    }
    if (cap > 0xffffffffull) return ss_fail(ctx, SS_ERR_CAPACITY, "too many tile overlaps (%llu)", (unsigned long long)cap);
    b.pairs = (int64_t)cap;
    const int64_t pa = cap > 0 ? (int64_t)cap : 1;
    b.pkeys = SS_SCRATCH(ctx, uint32_t, pa);
    b.pvals = SS_SCRATCH(ctx, uint32_t, pa);
    uint32_t* pk2 = SS_SCRATCH(ctx, uint32_t, pa);
    uint32_t* pv2 = SS_SCRATCH(ctx, uint32_t, pa);
    if (!b.pkeys || !b.pvals || !pk2 || !pv2) return SS_ERR_CUDA;
    SS_CUDA(ctx, ss_launch((k_clamp_pairs), dim3(1), dim3(1), 0, s, (const uint64_t*)total, cap, b.n_pairs, status));
    SS_CHECK_LAUNCH(ctx);
    if (cap > 0) {
        ss_tic(ctx, KC_BIN);
        SS_CUDA(ctx, ss_launch((k_emit_warp<R>), dim3(gridn(ctx, n)), dim3(256), 0, s, (const SplatRec<R>*)b.rec, b.dvals, b.rcnt, b.roff, n,
                               b.tiles_x, b.pkeys, b.pvals, b.roffj, cap));
        SS_CHECK_LAUNCH(ctx);
        ss_toc(ctx, KC_BIN);
        ss_tic(ctx, KC_TILE_SORT);
        SS_TRY(ss_radix_sort_u32(ctx, b.pkeys, b.pvals, pk2, pv2, (int64_t)cap, b.tile_bits, b.n_pairs));
        ss_toc(ctx, KC_TILE_SORT);
        ss_tic(ctx, KC_BIN);
        SS_CUDA(ctx, ss_launch((k_ranges), dim3(gridn(ctx, (int64_t)cap)), dim3(256), 0, s, b.pkeys, (const uint64_t*)b.n_pairs, b.ranges));
        SS_CHECK_LAUNCH(ctx);
        ss_toc(ctx, KC_BIN);
    }
    return SS_OK;
}

template <typename R>
int build_bins(ss_ctx* ctx, const ss_model* m, const ss_camera* cam, const ss_light* L, const ss_render_opts* o,
               Bins& b, DebugOut* dbg) {
    cudaStream_t s = ctx->stream;
    b.n_in = o->subset ? o->subset_count : m->count;
    b.tiles_x = (cam->width + TILE - 1) / TILE;
    b.tiles_y = (cam->height + TILE - 1) / TILE;
    b.n_tiles = b.tiles_x * b.tiles_y;
    b.tile_bits = 1;
    while ((1 << b.tile_bits) < b.n_tiles) ++b.tile_bits;
    const int64_t n = b.n_in;
    const int64_t na = n > 0 ? n : 1;
    b.dkey64 = SS_SCRATCH(ctx, uint64_t, na);
    b.dkeys = SS_SCRATCH(ctx, uint32_t, na);
    unsigned long long* kminmax = SS_SCRATCH(ctx, unsigned long long, 2);
    b.dvals = SS_SCRATCH(ctx, uint32_t, na);
    uint32_t* kalt = SS_SCRATCH(ctx, uint32_t, na);
    uint32_t* valt = SS_SCRATCH(ctx, uint32_t, na);
    b.mu = SS_SCRATCH(ctx, double2, na);
    b.roffj = SS_SCRATCH(ctx, uint64_t, na);
    b.roff = SS_SCRATCH(ctx, uint64_t, na);
    b.rcnt = SS_SCRATCH(ctx, uint32_t, na);
    b.rinv = SS_SCRATCH(ctx, uint32_t, na);
    b.rec = ss_scratch(ctx, sizeof(SplatRec<R>) * na);
    b.ranges = SS_SCRATCH(ctx, uint2, b.n_tiles);
    if (!b.dkey64 || !kminmax || !b.dkeys || !b.dvals || !kalt || !valt || !b.mu || !b.roffj || !b.roff || !b.rcnt || !b.rinv || !b.rec || !b.ranges)
        return SS_ERR_CUDA;
    SS_CUDA(ctx, cudaMemsetAsync(b.ranges, 0, sizeof(uint2) * b.n_tiles, s));
    DebugOut none;
    memset(&none, 0, sizeof(none));
    if (n > 0) {
        ss_tic(ctx, KC_PREPROCESS);
        SS_CUDA(ctx, ss_launch((k_init_minmax), dim3(1), dim3(1), 0, s, kminmax));
        SS_CHECK_LAUNCH(ctx);
#define SS_PRE(DEG)                                                                                      \
    SS_CUDA(ctx, ss_launch((k_preprocess<DEG, R, PT>), dim3(gridn(ctx, n, 128)), dim3(128), 0, s, *m, *cam, *L, o->subset, n, o->extent_cutoff, b.dkey64, \
                                                         b.dvals, (SplatRec<R>*)b.rec, b.mu, dbg ? *dbg : none,  \
                                                         kminmax))
#define SS_PRE_ALL()              \
    switch (m->sh_degree) {       \
        case 0: SS_PRE(0); break; \
        case 1: SS_PRE(1); break; \
        case 2: SS_PRE(2); break; \
        default: SS_PRE(3); break; \
    }
        bool f64p = false;  // float64 parameter columns: the fp64 instantiation only
        if constexpr (sizeof(R) == 8) {
            f64p = m->param_dtype == 1;
            if (f64p) {
                using PT = double;
                SS_PRE_ALL();
            }
        }
        if (!f64p) {
            using PT = float;
            SS_PRE_ALL();
        }
#undef SS_PRE_ALL
#undef SS_PRE
        SS_CHECK_LAUNCH(ctx);
        ss_toc(ctx, KC_PREPROCESS);
        ss_tic(ctx, KC_DEPTH_SORT);
        SS_CUDA(ctx, ss_launch((k_key32), dim3(gridn(ctx, n)), dim3(256), 0, s, b.dkey64, n, kminmax, b.dkeys));
        SS_CHECK_LAUNCH(ctx);
        SS_TRY(ss_radix_sort_u32(ctx, b.dkeys, b.dvals, kalt, valt, n, 32));
        SS_CUDA(ctx, ss_launch((k_fix_ties), dim3(gridn(ctx, n)), dim3(256), 0, s, b.dkeys, b.dvals, b.dkey64, n));
        SS_CHECK_LAUNCH(ctx);
        ss_toc(ctx, KC_DEPTH_SORT);
    }
    return bin_pairs<R>(ctx, b, o->bins_status);
}

template <typename R>
int forward(ss_ctx* ctx, const ss_camera* cam, const ss_render_opts* o, const Bins& b, R* img, R* T,
            uint32_t* tile_stop) {
    ss_tic(ctx, KC_FORWARD);
    uint32_t* order = SS_SCRATCH(ctx, uint32_t, b.n_tiles);
    if (!order) return SS_ERR_CUDA;
    const bool hint = o->tile_hint && o->tile_hint_len == b.n_tiles;
    if (hint && o->tile_order && o->tile_order_valid) {
        order = o->tile_order;  // the previous backward's order = the order of this hint
    } else {
        SS_CUDA(ctx, ss_launch((k_tile_order), dim3(1), dim3(1024), 0, ctx->stream, b.ranges, hint ? o->tile_hint : nullptr, b.n_tiles,
                               order));
        SS_CHECK_LAUNCH(ctx);
    }
    if constexpr (sizeof(R) == 4) {
        const bool count = ss_timing_on(ctx);
        SS_CUDA(ctx, ss_launch(count ? k_blend_fwd2<true> : k_blend_fwd2<false>, dim3((b.n_tiles + WPB - 1) / WPB), dim3(32 * WPB), 0, ctx->stream,
            b.ranges, b.pvals, b.mu, (const SplatRec<float>*)b.rec, cam->width, cam->height, b.tiles_x, b.n_tiles,
            o->background[0], o->background[1], o->background[2], img, T, tile_stop,
            count ? ctx->dev_counters : nullptr, order));
    }
    else
        SS_CUDA(ctx, ss_launch((k_blend_fwd<R>), dim3((b.n_tiles + WPB - 1) / WPB), dim3(32 * WPB), 0, ctx->stream, 
            b.ranges, b.pvals, b.mu, (const SplatRec<R>*)b.rec, cam->width, cam->height, b.tiles_x, b.n_tiles,
            o->background[0], o->background[1], o->background[2], img, T, tile_stop,
            ss_timing_on(ctx) ? ctx->dev_counters : nullptr, order));
    SS_CHECK_LAUNCH(ctx);
    ss_toc(ctx, KC_FORWARD);
    return SS_OK;
}

template <typename R>
int render_t(ss_ctx* ctx, const ss_model* m, const ss_camera* cam, const ss_light* L, const ss_render_opts* o,
             void* img, void* T, ss_render_stats* st) {
    Bins b;
    SS_TRY(build_bins<R>(ctx, m, cam, L, o, b, nullptr));
    SS_TRY(forward<R>(ctx, cam, o, b, (R*)img, (R*)T, nullptr));
    if (st) {
        st->visible = -1;
        st->pairs = b.pairs;
        st->tiles = b.n_tiles;
    }
    return SS_OK;
}

// The chain rule of nv views (host ChainViews) over inputs [j0, j1) into a
// gradient layout of ld rows from row0 (see ss_chain_views_range); scratch
// from the current call's arena.  The per-view backward of the fp32 blend
// runs it with one view, so a view's gradient is the same kernel's whether
// the chain is deferred to the step or not (bit-identical by construction).
int launch_chain_views(ss_ctx* ctx, const ss_model* m, const ChainViews& hv, int nv, const int64_t* subset,
                       int64_t j0, int64_t j1, int64_t row0, int64_t rows, float* grad, int64_t ld, int init = 0) {
    cudaStream_t s = ctx->stream;
    float4* shrec = SS_SCRATCH(ctx, float4, 2 * ld * nv);
    if (!shrec) return SS_ERR_CUDA;
    // without a subset k_chain_views writes every (view, row) record of rows
    // [0, rows) (a zero one where the row is not visible); a subset leaves
    // the other rows' records to this clear
    if (subset) SS_CUDA(ctx, cudaMemsetAsync(shrec, 0, sizeof(float4) * 2 * (size_t)ld * nv, s));
    ss_tic(ctx, KC_CHAIN);
#define SS_CHAINV(DEG)                                                                                                     \
    do {                                                                                                                   \
        SS_CUDA(ctx, ss_launch((k_chain_views<DEG>), dim3(gridn(ctx, j1 - j0, CVB)), dim3(CVB), 0, s, *m, hv,              \
                               nv, subset, j0, j1, row0, ld, grad, shrec, init));                                          \
        SS_CHECK_LAUNCH(ctx);                                                                                              \
        SS_CUDA(ctx, ss_launch((k_sh_grad_rows<DEG>), dim3(gridn(ctx, rows, CVB)), dim3(CVB), 0, s, hv, nv,               \
                               (const float4*)shrec, rows, ld, grad + 11 * ld, init));                                    \
        SS_CHECK_LAUNCH(ctx);                                                                                              \
    } while (0)
    switch (m->sh_degree) {
        case 0: SS_CHAINV(0); break;
        case 1: SS_CHAINV(1); break;
        case 2: SS_CHAINV(2); break;
        default: SS_CHAINV(3); break;
    }
#undef SS_CHAINV
    ss_toc(ctx, KC_CHAIN);
    return SS_OK;
}

template <typename R>
int backward_t(ss_ctx* ctx, const ss_model* m, const ss_camera* cam, const ss_light* L, const ss_render_opts* o,
               const float* gt, float* grad, double* loss, void* img_out, ss_render_stats* st) {
    cudaStream_t s = ctx->stream;
    Bins b;
    SS_TRY(build_bins<R>(ctx, m, cam, L, o, b, nullptr));
    const int64_t npx = (int64_t)cam->width * cam->height;
    const bool atomic = o->deterministic == 0;
    const bool chain = b.n_in > 0 && m->active_count > 0;
    R* img = img_out ? (R*)img_out : SS_SCRATCH(ctx, R, 3 * npx);
    uint32_t* stop = SS_SCRATCH(ctx, uint32_t, b.n_tiles);
    double* tloss = SS_SCRATCH(ctx, double, b.n_tiles);
    // per input row: the 9 screen-space sums (the deferred buffer, or scratch)
    R* g9 = (o->defer_g9 && sizeof(R) == 4) ? (R*)o->defer_g9 : SS_SCRATCH(ctx, R, 9 * (b.n_in > 0 ? b.n_in : 1));
    R* partials = atomic ? nullptr : SS_SCRATCH(ctx, R, 9 * (b.pairs > 0 ? b.pairs : 1));
    if (!img || !stop || !tloss || !g9 || (!atomic && !partials)) return SS_ERR_CUDA;
    if (atomic && b.n_in > 0) SS_CUDA(ctx, cudaMemsetAsync(g9, 0, sizeof(R) * 9 * (size_t)b.n_in, s));
    SS_TRY(forward<R>(ctx, cam, o, b, img, (R*)nullptr, stop));
    if (o->tile_hint && o->tile_hint_len == b.n_tiles)  // this call's walk lengths order the next forward
        SS_CUDA(ctx, cudaMemcpyAsync(o->tile_hint, stop, sizeof(uint32_t) * b.n_tiles, cudaMemcpyDeviceToDevice, s));
    const double inv_npx = 1.0 / (double)(3 * npx);
    if (o->gt_ready) SS_CUDA(ctx, cudaStreamWaitEvent(s, (cudaEvent_t)o->gt_ready, 0));
    ss_tic(ctx, KC_BACKWARD);
    uint32_t* order = SS_SCRATCH(ctx, uint32_t, b.n_tiles);
    if (!order) return SS_ERR_CUDA;
    SS_CUDA(ctx, ss_launch((k_tile_order), dim3(1), dim3(1024), 0, s, b.ranges, stop, b.n_tiles, order));
    SS_CHECK_LAUNCH(ctx);
    if (o->tile_order && o->tile_hint && o->tile_hint_len == b.n_tiles)  // reused by the next forward of this camera
        SS_CUDA(ctx, cudaMemcpyAsync(o->tile_order, order, sizeof(uint32_t) * b.n_tiles, cudaMemcpyDeviceToDevice, s));
#ifndef SS_BWD_PACKED
#define SS_BWD_PACKED 0  // measured (bench step, 8 views): packed 9.69 / scalar 9.21 ms -- 17 % fewer
#endif                   // instructions, but 114 registers drop issue-active from 77 % to 59 %
    const dim3 grid((b.n_tiles + WPB_BWD - 1) / WPB_BWD), block(32 * WPB_BWD);
    if (atomic)
        SS_CUDA(ctx, ss_launch((k_blend_bwd<R, true>), grid, block, 0, s, b.ranges, b.pvals, b.mu, (const SplatRec<R>*)b.rec,
                               b.roffj, stop, cam->width, cam->height, b.tiles_x, b.n_tiles, img, gt, (double)(3 * npx), g9,
                               tloss, order, (uint64_t)b.pairs));
    else if (sizeof(R) == 4 && SS_BWD_PACKED)
        SS_CUDA(ctx, ss_launch((k_blend_bwd2), grid, block, 0, s, b.ranges, b.pvals, b.mu, (const SplatRec<float>*)b.rec,
                               b.roffj, stop, cam->width, cam->height, b.tiles_x, b.n_tiles, (const float*)img, gt,
                               (double)(3 * npx), (float*)partials, tloss, order, (uint64_t)b.pairs));
    else
        SS_CUDA(ctx, ss_launch((k_blend_bwd<R, false>), grid, block, 0, s, b.ranges, b.pvals, b.mu, (const SplatRec<R>*)b.rec,
                               b.roffj, stop, cam->width, cam->height, b.tiles_x, b.n_tiles, img, gt, (double)(3 * npx),
                               partials, tloss, order, (uint64_t)b.pairs));
    SS_CHECK_LAUNCH(ctx);
    SS_CUDA(ctx, ss_launch((k_loss_reduce), dim3(1), dim3(256), 0, s, tloss, b.n_tiles, inv_npx, loss));
    SS_CHECK_LAUNCH(ctx);
    ss_toc(ctx, KC_BACKWARD);
    if (chain && !atomic) {  // fixed-order sum of each splat's per-tile partials
        ss_tic(ctx, KC_CHAIN);
        SS_CUDA(ctx, ss_launch((k_sum_partials<R>), dim3(gridn(ctx, b.n_in)), dim3(256), 0, s, b.roff, b.rcnt, b.dvals,
                               partials, (const SplatRec<R>*)b.rec, b.n_in, g9, (uint64_t)b.pairs));
        SS_CHECK_LAUNCH(ctx);
        ss_toc(ctx, KC_CHAIN);
    }
    if (chain && o->defer_g9 && sizeof(R) == 4) {  // chain rule left to ss_chain_views
        SS_CUDA(ctx, cudaMemcpyAsync(o->defer_rinv, b.rinv, sizeof(uint32_t) * (size_t)b.n_in, cudaMemcpyDeviceToDevice, s));
    } else if (chain && sizeof(R) == 4) {
        ChainViews hv;
        memset(&hv, 0, sizeof(hv));
        hv.cam[0] = *cam;
        hv.light[0] = *L;
        hv.g9[0] = (const float*)g9;
        hv.rinv[0] = b.rinv;
        const int64_t a = m->active_count;
        SS_TRY(launch_chain_views(ctx, m, hv, 1, o->subset, 0, b.n_in, 0, a, grad, a));
    } else if (chain) {
        ss_tic(ctx, KC_CHAIN);
        float4* shrec = SS_SCRATCH(ctx, float4, 2 * (int64_t)m->active_count);
        if (!shrec) return SS_ERR_CUDA;
        SS_CUDA(ctx, cudaMemsetAsync(shrec, 0, sizeof(float4) * 2 * (size_t)m->active_count, s));
#define SS_CHAIN(DEG)                                                                                     \
    SS_CUDA(ctx, ss_launch((k_chain<R, DEG, PT>), dim3(gridn(ctx, b.n_in, 128)), dim3(128), 0, s, *m, *cam, *L, o->subset, b.rinv, g9, b.n_in,        \
                                                            o->extent_cutoff, grad, shrec));                      \
    SS_CUDA(ctx, ss_launch((k_sh_grad<DEG>), dim3((unsigned)(((int64_t)m->active_count + SHG_ROWS - 1) / SHG_ROWS)), dim3(256), 0, s,              \
        *L, shrec, m->active_count, grad + 11 * (int64_t)m->active_count))
#define SS_CHAIN_ALL()              \
    switch (m->sh_degree) {         \
        case 0: SS_CHAIN(0); break; \
        case 1: SS_CHAIN(1); break; \
        case 2: SS_CHAIN(2); break; \
        default: SS_CHAIN(3); break; \
    }
        bool f64p = false;
        if constexpr (sizeof(R) == 8) {
            f64p = m->param_dtype == 1;
            if (f64p) {
                using PT = double;
                SS_CHAIN_ALL();
            }
        }
        if (!f64p) {
            using PT = float;
            SS_CHAIN_ALL();
        }
#undef SS_CHAIN_ALL
#undef SS_CHAIN
        SS_CHECK_LAUNCH(ctx);
        ss_toc(ctx, KC_CHAIN);
    }
    if (st) {
        st->visible = -1;
        st->pairs = b.pairs;
        st->tiles = b.n_tiles;
    }
    return SS_OK;
}

// the rest of PreparedSplats (ss_prepare_extras), one thread per prepared splat
template <int DEG, typename PT>
__global__ void k_prepare_extras(ss_model m, ss_camera cam, ss_light L, const int64_t* __restrict__ rows, int64_t M,
                                 ss_prepared_extras o) {
    SS_PDL_WAIT();
    constexpr int B = ss_sh_bases(DEG);
    const ParamView<PT> pv(m);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = rows[i];
        Proj P;
        ss_cam_point(cam, pv.means + row * 3, P.d, P.mc);
        const PT* ls = pv.ls + row * 3;
        ss_project(cam, ls, pv.quats + row * 4, true, P);
        PT shv[3 * B];
        ss_load_sh<DEG, PT>(pv.sh + row * 3 * B, shv);
        Shade<DEG, double> S;
        ss_shade_v<DEG, double, PT>(L, ls, shv, pv.vis[row], P.d, P.Rq, S);
        if (o.mu_cam) for (int k = 0; k < 3; ++k) o.mu_cam[3 * i + k] = P.mc[k];
        if (o.J) for (int r = 0; r < 2; ++r) for (int k = 0; k < 3; ++k) o.J[6 * i + 3 * r + k] = P.J[r][k];
        if (o.sigma3d)
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b)
                    o.sigma3d[9 * i + 3 * a + b] = da(da(dm(dm(P.Rq[a][0], P.S2[0]), P.Rq[b][0]), dm(dm(P.Rq[a][1], P.S2[1]), P.Rq[b][1])),
                                                      dm(dm(P.Rq[a][2], P.S2[2]), P.Rq[b][2]));
        if (o.cov_cam) for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) o.cov_cam[9 * i + 3 * a + b] = P.cov[a][b];
        if (o.view_dir) for (int k = 0; k < 3; ++k) o.view_dir[3 * i + k] = S.vdir[k];
        if (o.view_dist) o.view_dist[i] = S.dist;
        if (o.n_hat) for (int k = 0; k < 3; ++k) o.n_hat[3 * i + k] = S.nhat[k];
        if (o.n_axis) o.n_axis[i] = S.axis;
        if (o.Y) for (int b = 0; b < B; ++b) o.Y[B * i + b] = S.Y[b];
        if (o.albedo_est) for (int c = 0; c < 3; ++c) o.albedo_est[3 * i + c] = S.albedo[c];
        if (o.cos) o.cos[i] = S.cosv;
        if (o.vis) o.vis[i] = S.vis;
    }
}

// composite() of prepared splats already in draw order (ss_composite)
__global__ void k_prep_recs(int64_t n, const double* __restrict__ mu2d, const double* __restrict__ inv2d,
                            const double* __restrict__ opacity, const double* __restrict__ color,
                            const int32_t* __restrict__ windows, SplatRec<double>* __restrict__ rec, double2* __restrict__ mu,
                            uint64_t* __restrict__ dkey64, uint32_t* __restrict__ dvals) {
    SS_PDL_WAIT();
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        SplatRec<double> g;
        for (int k = 0; k < 4; ++k) g.win[k] = windows[4 * j + k];
        g.a = inv2d[3 * j];
        g.b = inv2d[3 * j + 1];
        g.c = inv2d[3 * j + 2];
        g.o = opacity[j];
        for (int c = 0; c < 3; ++c) g.col[c] = color[3 * j + c];
        rec[j] = g;
        mu[j] = make_double2(mu2d[2 * j], mu2d[2 * j + 1]);
        dkey64[j] = 0;            // visible
        dvals[j] = (uint32_t)j;   // rank = position in the draw order
    }
}

__global__ void k_order_out(const uint64_t* dkey64, const uint32_t* dvals, const uint64_t* vpos, int64_t n,
                            int64_t* order) {
    SS_PDL_WAIT();
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        if (dkey64[dvals[r]] != ~0ull) order[r] = (int64_t)vpos[dvals[r]];
}

__global__ void k_debug_bins(const Bins b, int64_t* order_rows, const int64_t* subset, int64_t* ranges_out,
                             int64_t* pair_rank) {
    SS_PDL_WAIT();
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = tid; r < b.n_in; r += nt)
        if (order_rows && b.dkey64[b.dvals[r]] != ~0ull) order_rows[r] = subset ? subset[b.dvals[r]] : (int64_t)b.dvals[r];
    for (int64_t t = tid; t < b.n_tiles; t += nt)
        if (ranges_out) {
            ranges_out[2 * t] = b.ranges[t].x;
            ranges_out[2 * t + 1] = b.ranges[t].y;
        }
    for (int64_t p = tid; p < b.pairs; p += nt)
        if (pair_rank) pair_rank[p] = b.rinv[b.pvals[p]];
}

}  // namespace

extern "C" {

int ss_render(ss_ctx* ctx, const ss_model* m, const ss_camera* cam, const ss_light* L, const ss_render_opts* o,
              void* img, void* T, ss_render_stats* st) {
    SS_NVTX("ss_render");
    if (!ctx) return SS_ERR_INVALID;
    SS_TRY(validate(ctx, m, cam, o));
    if (!img) return ss_fail(ctx, SS_ERR_INVALID, "image_out is required");
    SS_TRY(ss_scratch_reset(ctx));
    return o->precision ? render_t<double>(ctx, m, cam, L, o, img, T, st) : render_t<float>(ctx, m, cam, L, o, img, T, st);
}

int ss_backward(ss_ctx* ctx, const ss_model* m, const ss_camera* cam, const ss_light* L, const ss_render_opts* o,
                const float* gt, float* grad, double* loss, void* img, ss_render_stats* st) {
    SS_NVTX("ss_backward");
    if (!ctx) return SS_ERR_INVALID;
    SS_TRY(validate(ctx, m, cam, o));
    if (!gt || !grad || !loss) return ss_fail(ctx, SS_ERR_INVALID, "gt, grad_accum and loss_accum are required");
    if (o->defer_g9 && (o->precision || !o->defer_rinv))
        return ss_fail(ctx, SS_ERR_INVALID, "defer_g9 needs the fp32 blend and defer_rinv");
    SS_TRY(ss_scratch_reset(ctx));
    return o->precision ? backward_t<double>(ctx, m, cam, L, o, gt, grad, loss, img, st)
                        : backward_t<float>(ctx, m, cam, L, o, gt, grad, loss, img, st);
}

int ss_composite(ss_ctx* ctx, int64_t n, const double* mu2d, const double* inv2d, const double* opacity, const double* color,
                 const int32_t* windows, int32_t width, int32_t height, const double* background, double* img, double* T) {
    if (!ctx || !img || !background || width < 1 || height < 1 || n < 0) return SS_ERR_INVALID;
    if (n > 0 && (!mu2d || !inv2d || !opacity || !color || !windows)) return SS_ERR_INVALID;
    if (n > 0xffffffffll) return ss_fail(ctx, SS_ERR_CAPACITY, "too many splats");
    SS_TRY(ss_scratch_reset(ctx));
    cudaStream_t s = ctx->stream;
    Bins b;
    memset(&b, 0, sizeof(b));
    b.n_in = n;
    b.tiles_x = (width + TILE - 1) / TILE;
    b.tiles_y = (height + TILE - 1) / TILE;
    b.n_tiles = b.tiles_x * b.tiles_y;
    b.tile_bits = 1;
    while ((1 << b.tile_bits) < b.n_tiles) ++b.tile_bits;
    const int64_t na = n > 0 ? n : 1;
    b.dkey64 = SS_SCRATCH(ctx, uint64_t, na);
    b.dvals = SS_SCRATCH(ctx, uint32_t, na);
    b.mu = SS_SCRATCH(ctx, double2, na);
    b.roffj = SS_SCRATCH(ctx, uint64_t, na);
    b.roff = SS_SCRATCH(ctx, uint64_t, na);
    b.rcnt = SS_SCRATCH(ctx, uint32_t, na);
    b.rinv = SS_SCRATCH(ctx, uint32_t, na);
    b.rec = ss_scratch(ctx, sizeof(SplatRec<double>) * na);
    b.ranges = SS_SCRATCH(ctx, uint2, b.n_tiles);
    uint32_t* stop = SS_SCRATCH(ctx, uint32_t, b.n_tiles);
    if (!b.dkey64 || !b.dvals || !b.mu || !b.roffj || !b.roff || !b.rcnt || !b.rinv || !b.rec || !b.ranges || !stop)
        return SS_ERR_CUDA;
    SS_CUDA(ctx, cudaMemsetAsync(b.ranges, 0, sizeof(uint2) * b.n_tiles, s));
    if (n > 0) {
        SS_CUDA(ctx, ss_launch((k_prep_recs), dim3(gridn(ctx, n)), dim3(256), 0, s, n, mu2d, inv2d, opacity, color, windows,
                               (SplatRec<double>*)b.rec, b.mu, b.dkey64, b.dvals));
        SS_CHECK_LAUNCH(ctx);
    }
    SS_TRY(bin_pairs<double>(ctx, b, nullptr));
    ss_camera cam;
    memset(&cam, 0, sizeof(cam));
    cam.width = width;
    cam.height = height;
    ss_render_opts o;
    memset(&o, 0, sizeof(o));
    for (int k = 0; k < 3; ++k) o.background[k] = background[k];
    return forward<double>(ctx, &cam, &o, b, img, T, stop);
}

int ss_chain_views_range(ss_ctx* ctx, const ss_model* m, const ss_camera* cams, const ss_light* lights,
                         int32_t n_views, const float* const* g9, const uint32_t* const* rinv, const int64_t* subset,
                         int64_t j0, int64_t j1, int64_t row0, int64_t rows, float* grad, int64_t ld) {
    return ss_chain_views_range_init(ctx, m, cams, lights, n_views, g9, rinv, subset, j0, j1, row0, rows, grad, ld, 0);
}

int ss_chain_views_range_init(ss_ctx* ctx, const ss_model* m, const ss_camera* cams, const ss_light* lights,
                              int32_t n_views, const float* const* g9, const uint32_t* const* rinv,
                              const int64_t* subset, int64_t j0, int64_t j1, int64_t row0, int64_t rows, float* grad,
                              int64_t ld, int32_t init) {
    SS_NVTX("ss_chain_views");
    if (!ctx || !m || !cams || !lights || !g9 || !rinv || !grad) return SS_ERR_INVALID;
    if (init && (subset || j0 != row0 || j1 < row0 + rows))
        return ss_fail(ctx, SS_ERR_INVALID, "init needs the whole row range without a subset");
    if (n_views < 1 || n_views > CV_MAX_VIEWS) return ss_fail(ctx, SS_ERR_INVALID, "1..%d views", CV_MAX_VIEWS);
    if (m->sh_degree < 0 || m->sh_degree > 3 || j0 < 0 || j1 < j0) return ss_fail(ctx, SS_ERR_INVALID, "bad model or row range");
    if (row0 < 0 || rows < 0 || ld < rows || row0 + rows > m->active_count)
        return ss_fail(ctx, SS_ERR_INVALID, "bad gradient layout (row0 %lld, rows %lld, ld %lld)", (long long)row0,
                       (long long)rows, (long long)ld);
    if (m->param_dtype != 0) return ss_fail(ctx, SS_ERR_INVALID, "the deferred chain rule takes float32 parameters");
    if (rows == 0 || j1 == j0) return SS_OK;
    SS_TRY(ss_scratch_reset(ctx));
    ChainViews hv;
    memset(&hv, 0, sizeof(hv));
    for (int v = 0; v < n_views; ++v) {
        if (!g9[v] || !rinv[v]) return ss_fail(ctx, SS_ERR_INVALID, "view %d: missing deferred buffers", v);
        hv.cam[v] = cams[v];
        hv.light[v] = lights[v];
        hv.g9[v] = g9[v];
        hv.rinv[v] = rinv[v];
    }
    return launch_chain_views(ctx, m, hv, n_views, subset, j0, j1, row0, rows, grad, ld, init);
}

int ss_chain_views(ss_ctx* ctx, const ss_model* m, const ss_camera* cams, const ss_light* lights, int32_t n_views,
                   const float* const* g9, const uint32_t* const* rinv, const int64_t* subset, int64_t n_in,
                   float* grad) {
    if (!m) return SS_ERR_INVALID;
    const int64_t a = m->active_count;
    if (a <= 0 || n_in <= 0) return SS_OK;
    return ss_chain_views_range(ctx, m, cams, lights, n_views, g9, rinv, subset, 0, n_in, 0, a, grad, a);
}

// loss = ((x[0] + x[1]) + x[2]) + ...: the reference's per-view loss sum order (optim.py:366-367)
__global__ void k_sum_f64_seq(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
    SS_PDL_WAIT();
    double t = 0.0;
    for (int64_t i = 0; i < n; ++i) t += x[i];
    *out = t;
}

int ss_sum_f64(ss_ctx* ctx, const double* x, int64_t n, double* out) {
    if (!ctx || !x || !out || n < 0) return SS_ERR_INVALID;
    SS_CUDA(ctx, ss_launch((k_sum_f64_seq), dim3(1), dim3(1), 0, ctx->stream, x, n, out));
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}

int ss_prepare_splats(ss_ctx* ctx, const ss_model* m, const ss_camera* cam, const ss_light* L,
                      const ss_render_opts* o, ss_prepared* out, int64_t* visible_out) {
    if (!ctx) return SS_ERR_INVALID;
    SS_TRY(validate(ctx, m, cam, o));
    if (!out) return ss_fail(ctx, SS_ERR_INVALID, "out is required");
    SS_TRY(ss_scratch_reset(ctx));
    cudaStream_t s = ctx->stream;
    const int64_t n = o->subset ? o->subset_count : m->count;
    const int64_t na = n > 0 ? n : 1;
    uint8_t* flag = SS_SCRATCH(ctx, uint8_t, na);
    uint64_t* vpos = SS_SCRATCH(ctx, uint64_t, na);
    uint64_t* vtot = SS_SCRATCH(ctx, uint64_t, 1);
    if (!flag || !vpos || !vtot) return SS_ERR_CUDA;
    if (n > 0) {
        if (m->param_dtype == 1)
            SS_CUDA(ctx, ss_launch((k_visible_flags<double>), dim3(gridn(ctx, n)), dim3(256), 0, s, *m, *cam, o->subset, n, flag));
        else
            SS_CUDA(ctx, ss_launch((k_visible_flags<float>), dim3(gridn(ctx, n)), dim3(256), 0, s, *m, *cam, o->subset, n, flag));
        SS_CHECK_LAUNCH(ctx);
    }
    SS_TRY(ss_scan_u8_to_u64(ctx, flag, vpos, n, vtot));
    uint64_t M = 0;
    SS_TRY(ss_read_u64(ctx, vtot, &M));
    if ((int64_t)M > out->capacity) return ss_fail(ctx, SS_ERR_CAPACITY, "prepared capacity %lld < visible %llu",
                                                   (long long)out->capacity, (unsigned long long)M);
    DebugOut dbg;
    dbg.p = *out;
    dbg.vpos = vpos;
    Bins b;
    SS_TRY(build_bins<double>(ctx, m, cam, L, o, b, &dbg));
    if (out->order && n > 0) {
        SS_CUDA(ctx, ss_launch((k_order_out), dim3(gridn(ctx, n)), dim3(256), 0, s, b.dkey64, b.dvals, vpos, n, out->order));
        SS_CHECK_LAUNCH(ctx);
    }
    if (visible_out) *visible_out = (int64_t)M;
    SS_CUDA(ctx, ss_stream_sync(ctx));
    return SS_OK;
}

int ss_debug_bwd_stats(ss_ctx* ctx, unsigned long long out[8], int reset) {
    if (!ctx || !out) return SS_ERR_INVALID;
#ifdef SS_BWD_STATS
    SS_CUDA(ctx, ss_stream_sync(ctx));
    SS_CUDA(ctx, cudaMemcpyFromSymbol(out, g_bwd_stats, sizeof(unsigned long long) * 8));
    if (reset) {
        unsigned long long z[8] = {};
        SS_CUDA(ctx, cudaMemcpyToSymbol(g_bwd_stats, z, sizeof(z)));
    }
    return SS_OK;
#else
    (void)reset;
    return ss_fail(ctx, SS_ERR_INVALID, "built without SS_BWD_STATS");
#endif
}

int ss_prepare_extras(ss_ctx* ctx, const ss_model* m, const ss_camera* cam, const ss_light* L, const int64_t* rows,
                      int64_t M, ss_prepared_extras* out) {
    if (!ctx || !m || !cam || !L || !out || (M > 0 && !rows)) return SS_ERR_INVALID;
    if (m->sh_degree < 0 || m->sh_degree > 3 || M < 0) return ss_fail(ctx, SS_ERR_INVALID, "bad model or count");
    if (M == 0) return SS_OK;
    SS_TRY(ss_scratch_reset(ctx));
#define SS_EXTRAS(DEG, PT) SS_CUDA(ctx, ss_launch((k_prepare_extras<DEG, PT>), dim3(gridn(ctx, M)), dim3(256), 0, ctx->stream, \
                                                   *m, *cam, *L, rows, M, *out))
    if (m->param_dtype == 1) {
        switch (m->sh_degree) {
            case 0: SS_EXTRAS(0, double); break;
            case 1: SS_EXTRAS(1, double); break;
            case 2: SS_EXTRAS(2, double); break;
            default: SS_EXTRAS(3, double); break;
        }
    } else {
        switch (m->sh_degree) {
            case 0: SS_EXTRAS(0, float); break;
            case 1: SS_EXTRAS(1, float); break;
            case 2: SS_EXTRAS(2, float); break;
            default: SS_EXTRAS(3, float); break;
        }
    }
#undef SS_EXTRAS
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}

int ss_debug_bins(ss_ctx* ctx, const ss_model* m, const ss_camera* cam, const ss_render_opts* o, int64_t* order_rows,
                  int64_t rows_cap, int64_t* ranges_out, int64_t tiles_cap, int64_t* pair_rank, int64_t pairs_cap,
                  ss_render_stats* st) {
    if (!ctx) return SS_ERR_INVALID;
    SS_TRY(validate(ctx, m, cam, o));
    SS_TRY(ss_scratch_reset(ctx));
    ss_light L;
    memset(&L, 0, sizeof(L));
    L.direction[1] = -1.0;
    Bins b;
    SS_TRY(build_bins<float>(ctx, m, cam, &L, o, b, nullptr));
    if (b.n_in > rows_cap || b.n_tiles > tiles_cap || b.pairs > pairs_cap)
        return ss_fail(ctx, SS_ERR_CAPACITY, "debug output too small (rows %lld tiles %d pairs %lld)",
                       (long long)b.n_in, b.n_tiles, (long long)b.pairs);
    SS_CUDA(ctx, ss_launch((k_debug_bins), dim3(gridn(ctx, b.n_in > b.pairs ? b.n_in : b.pairs)), dim3(256), 0, ctx->stream, b, order_rows, o->subset,
                                                                                          ranges_out, pair_rank));
    SS_CHECK_LAUNCH(ctx);
    if (st) {
        st->visible = -1;
        st->pairs = b.pairs;
        st->tiles = b.n_tiles;
    }
    SS_CUDA(ctx, ss_stream_sync(ctx));
    return SS_OK;
}

}  // extern "C"
