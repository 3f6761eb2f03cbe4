// Differentiable tile rasterizer for the splatstream compositing rules.
//
//   K1  k_preprocess    per Gaussian: fp64 projection, Sigma2d, 3-sigma
//                       window, depth key, relit colour     (render.py:226-290)
//   K3a depth sort      stable radix sort of fp64-depth bits -> exact
//                       lexsort((rows, depth)) order         (render.py:283)
//   K2  k_count/k_emit  rank-ordered splat records, tile-overlap counts,
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
struct SplatRec {
    R a, b, c;      // inverse 2D covariance [[a, b], [b, c]]
    R o;            // opacity
    R col[3];       // clamped colour
    int win[4];     // x0, x1, y0, y1
};

struct PerG {      // per-Gaussian preprocess output (index j = position in the input rows)
    double mu[2];
    double a, b, c, o;
    double col[3];
    int win[4];
};

struct Bins {
    int64_t n_in;            // rows considered (subset or all)
    int64_t visible;
    int64_t pairs;
    int tiles_x, tiles_y, n_tiles, tile_bits;
    uint64_t* dkeys;         // [n_in] depth keys, sorted
    uint32_t* dvals;         // [n_in] input index j, sorted by depth
    PerG* perg;              // [n_in]
    double2* rmu;            // [n_in] rank-ordered mu2d
    uint64_t* roff;          // [n_in] rank -> first pair (pre-sort position)
    uint32_t* rcnt;          // [n_in] tiles touched
    void* rrec;              // [n_in] rank-ordered SplatRec<R>
    uint32_t* pkeys;         // [pairs] tile id (sorted)
    uint32_t* pvals;         // [pairs] rank (sorted)
    uint2* ranges;           // [n_tiles]
};

// ---------------------------------------------------------------- K1
struct DebugOut {
    ss_prepared p;
    const uint64_t* vpos;    // visible position of input j
};

__global__ void k_visible_flags(ss_model m, ss_camera cam, const int64_t* subset, int64_t n_in, uint8_t* flag) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_in; j += (int64_t)gridDim.x * blockDim.x) {
        int64_t row = subset ? subset[j] : j;
        double d[3], mc[3];
        ss_cam_point(cam, m.means + row * 3, d, mc);
        flag[j] = mc[2] >= cam.near_plane;
    }
}

__global__ void k_preprocess(ss_model m, ss_camera cam, ss_light L, const int64_t* __restrict__ subset, int64_t n_in,
                             int cutoff, uint64_t* __restrict__ dkeys, uint32_t* __restrict__ dvals,
                             PerG* __restrict__ perg, DebugOut dbg) {
    const int B = ss_sh_bases(m.sh_degree);
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_in; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = subset ? subset[j] : j;
        Proj P;
        ss_cam_point(cam, m.means + row * 3, P.d, P.mc);
        dvals[j] = (uint32_t)j;
        if (!(P.mc[2] >= cam.near_plane)) {
            dkeys[j] = ~0ull;
            continue;
        }
        dkeys[j] = (uint64_t)__double_as_longlong(P.mc[2]);  // z >= near > 0: bits order as the value
        ss_project(cam, m.log_scales + row * 3, m.quaternions + row * 4, cutoff != 0, P);
        Shade S;
        ss_shade(L, m.log_scales + row * 3, m.sh_coeffs + row * 3 * B, B, m.sh_degree, m.light_visibility[row], P.d,
                 P.Rq, S);
        PerG g;
        g.mu[0] = P.mu[0];
        g.mu[1] = P.mu[1];
        g.a = P.s11 / P.det;
        g.b = -P.s01 / P.det;
        g.c = P.s00 / P.det;
        g.o = 1.0 / (1.0 + exp(-(double)m.logit_opacities[row]));
        for (int c = 0; c < 3; ++c) g.col[c] = fmin(fmax(S.pre[c], 0.0), 1.0);
        ss_window(P, cam.width, cam.height, g.win);
        perg[j] = g;
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
}

// ---------------------------------------------------------------- K2
__device__ __forceinline__ void win_tiles(const int w[4], int& tx0, int& tx1, int& ty0, int& ty1) {
    tx0 = w[0] / TILE;
    tx1 = (w[1] - 1) / TILE;
    ty0 = w[2] / TILE;
    ty1 = (w[3] - 1) / TILE;
}

template <typename R>
__global__ void k_count(const uint64_t* __restrict__ dkeys, const uint32_t* __restrict__ dvals,
                        const PerG* __restrict__ perg, int64_t n_in, double2* __restrict__ rmu,
                        SplatRec<R>* __restrict__ rrec, uint32_t* __restrict__ rcnt) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_in; r += (int64_t)gridDim.x * blockDim.x) {
        if (dkeys[r] == ~0ull) {
            rcnt[r] = 0;
            continue;
        }
        const PerG g = perg[dvals[r]];
        rmu[r] = make_double2(g.mu[0], g.mu[1]);
        SplatRec<R> s;
        s.a = (R)g.a;
        s.b = (R)g.b;
        s.c = (R)g.c;
        s.o = (R)g.o;
        for (int c = 0; c < 3; ++c) s.col[c] = (R)g.col[c];
        for (int k = 0; k < 4; ++k) s.win[k] = g.win[k];
        rrec[r] = s;
        uint32_t cnt = 0;
        if (g.win[0] < g.win[1] && g.win[2] < g.win[3]) {
            int tx0, tx1, ty0, ty1;
            win_tiles(g.win, tx0, tx1, ty0, ty1);
            cnt = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
        }
        rcnt[r] = cnt;
    }
}

template <typename R>
__global__ void k_emit(const SplatRec<R>* __restrict__ rrec, const uint32_t* __restrict__ rcnt,
                       const uint64_t* __restrict__ roff, int64_t n_in, int tiles_x, uint32_t* __restrict__ pkeys,
                       uint32_t* __restrict__ pvals) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_in; r += (int64_t)gridDim.x * blockDim.x) {
        if (!rcnt[r]) continue;
        int tx0, tx1, ty0, ty1;
        win_tiles(rrec[r].win, tx0, tx1, ty0, ty1);
        uint64_t p = roff[r];
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx, ++p) {
                pkeys[p] = (uint32_t)(ty * tiles_x + tx);
                pvals[p] = (uint32_t)r;
            }
    }
}

__global__ void k_ranges(const uint32_t* __restrict__ keys, int64_t n, uint2* __restrict__ ranges) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t t = keys[s];
        if (s == 0 || keys[s - 1] != t) ranges[t].x = (uint32_t)s;
        if (s == n - 1 || keys[s + 1] != t) ranges[t].y = (uint32_t)(s + 1);
    }
}

// ---------------------------------------------------------------- blend math
template <typename R> __device__ __forceinline__ R ss_exp(R x);
template <> __device__ __forceinline__ float ss_exp<float>(float x) { return __expf(x); }
template <> __device__ __forceinline__ double ss_exp<double>(double x) { return exp(x); }

// Staged splat (shared memory).  For fp32 the centre is tile-relative
// (computed in fp64 then rounded) so dx keeps full precision; for fp64 it
// is absolute and dx = (px + 0.5) - mu exactly as the reference computes it.
template <typename R>
struct Staged {
    R mx, my, a, b, c, o, col0, col1, col2;
    int wx0, wx1, wy0, wy1;  // window in tile-local pixel coords, clipped to [0, 16]
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
    s.col0 = rec.col[0];
    s.col1 = rec.col[1];
    s.col2 = rec.col[2];
    s.wx0 = min(max(rec.win[0] - X0, 0), TILE);
    s.wx1 = min(max(rec.win[1] - X0, 0), TILE);
    s.wy0 = min(max(rec.win[2] - Y0, 0), TILE);
    s.wy1 = min(max(rec.win[3] - Y0, 0), TILE);
}

template <typename R>
__device__ __forceinline__ void pixel_delta(const Staged<R>& s, int lx, int ly, int X0, int Y0, R& dx, R& dy) {
    if (sizeof(R) == 4) {
        dx = ((R)lx + (R)0.5) - s.mx;
        dy = ((R)ly + (R)0.5) - s.my;
    } else {
        dx = ((R)(X0 + lx) + (R)0.5) - s.mx;
        dy = ((R)(Y0 + ly) + (R)0.5) - s.my;
    }
}

// ---------------------------------------------------------------- K5 forward
constexpr int FWD_THREADS = 256;

template <typename R>
__global__ void __launch_bounds__(FWD_THREADS) k_blend_fwd(const uint2* __restrict__ ranges,
                                                           const uint32_t* __restrict__ pvals,
                                                           const double2* __restrict__ rmu,
                                                           const SplatRec<R>* __restrict__ rrec, int W, int H,
                                                           int tiles_x, double bg0, double bg1, double bg2,
                                                           R* __restrict__ img, R* __restrict__ Tout,
                                                           uint32_t* __restrict__ tile_stop,
                                                           unsigned long long* __restrict__ eval_count) {
    __shared__ Staged<R> sm[FWD_THREADS];
    __shared__ int s_last;
    const int tile = blockIdx.x;
    const int X0 = (tile % tiles_x) * TILE, Y0 = (tile / tiles_x) * TILE;
    const int lx = threadIdx.x % TILE, ly = threadIdx.x / TILE;
    const int px = X0 + lx, py = Y0 + ly;
    const bool inside = px < W && py < H;
    const uint2 rg = ranges[tile];
    R T = 1, c0 = 0, c1 = 0, c2 = 0;
    bool done = !inside;
    int last = -1;
    uint32_t evals = 0;
    if (threadIdx.x == 0) s_last = -1;
    for (uint32_t b0 = rg.x; b0 < rg.y; b0 += FWD_THREADS) {
        if (__syncthreads_count(!done) == 0) break;
        const uint32_t i = b0 + threadIdx.x;
        if (i < rg.y) {
            const uint32_t r = pvals[i];
            stage(sm[threadIdx.x], rmu[r], rrec[r], X0, Y0);
        }
        __syncthreads();
        const int nb = min((uint32_t)FWD_THREADS, rg.y - b0);
        for (int k = 0; k < nb && !done; ++k) {
            const Staged<R>& s = sm[k];
            if (lx < s.wx0 || lx >= s.wx1 || ly < s.wy0 || ly >= s.wy1) continue;
            R dx, dy;
            pixel_delta(s, lx, ly, X0, Y0, dx, dy);
            const R power = (R)-0.5 * (s.a * dx * dx + (R)2 * s.b * dx * dy + s.c * dy * dy);
            const R alpha = min(s.o * ss_exp<R>(power), (R)ALPHA_CAP);
            const R w = alpha * T;
            c0 += w * s.col0;
            c1 += w * s.col1;
            c2 += w * s.col2;
            T = T * ((R)1 - alpha);
            last = (int)(b0 - rg.x) + k;
            ++evals;
            if (T < (R)T_CUTOFF) done = true;
        }
    }
    if (last >= 0) atomicMax(&s_last, last);
    if (eval_count) {
#pragma unroll
        for (int o = 16; o; o >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, o);
        if ((threadIdx.x & 31) == 0 && evals) atomicAdd(eval_count, (unsigned long long)evals);
    }
    __syncthreads();
    if (threadIdx.x == 0 && tile_stop) tile_stop[tile] = (uint32_t)(s_last + 1);
    if (inside) {
        const int64_t p = (int64_t)py * W + px;
        img[3 * p + 0] = c0 + T * (R)bg0;
        img[3 * p + 1] = c1 + T * (R)bg1;
        img[3 * p + 2] = c2 + T * (R)bg2;
        if (Tout) Tout[p] = T;
    }
}

// ---------------------------------------------------------------- K6 backward
constexpr int BWD_THREADS = 64;   // 4 pixels per thread: (lx, ly0 + 4 q)
constexpr int BWD_PPT = 4;
constexpr int BWD_BATCH = 64;
constexpr int BWD_WARPS = BWD_THREADS / 32;

// Transposed butterfly: reduces v[0..7] over the warp with 7+2 shuffles;
// lane l with (l & 3) == 0 ends with the sum of value index
// 4*bit4(l) + 2*bit3(l) + bit2(l).
template <typename R>
__device__ __forceinline__ R warp_reduce8(R v[8], int lane) {
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

template <typename R>
__global__ void __launch_bounds__(BWD_THREADS) k_blend_bwd(const uint2* __restrict__ ranges,
                                                           const uint32_t* __restrict__ pvals,
                                                           const double2* __restrict__ rmu,
                                                           const SplatRec<R>* __restrict__ rrec,
                                                           const uint64_t* __restrict__ roff,
                                                           const uint32_t* __restrict__ tile_stop, int W, int H,
                                                           int tiles_x, const R* __restrict__ img,
                                                           const float* __restrict__ gt, double npx3,
                                                           R* __restrict__ partials, double* __restrict__ tile_loss) {
    __shared__ Staged<R> sm[BWD_BATCH];
    __shared__ uint64_t s_pidx[BWD_BATCH];
    __shared__ R s_red[BWD_WARPS][BWD_BATCH][9];
    __shared__ double s_loss[BWD_WARPS];
    const int tile = blockIdx.x;
    const int X0 = (tile % tiles_x) * TILE, Y0 = (tile / tiles_x) * TILE;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = threadIdx.x % TILE, ly0 = threadIdx.x / TILE;
    const uint2 rg = ranges[tile];
    const uint32_t stop = rg.x + (tile_stop ? min(tile_stop[tile], rg.y - rg.x) : (rg.y - rg.x));

    R T[BWD_PPT], pre[BWD_PPT][3], C[BWD_PPT][3], gC[BWD_PPT][3];
    bool dn[BWD_PPT];
    double loss = 0.0;
#pragma unroll
    for (int q = 0; q < BWD_PPT; ++q) {
        const int ly = ly0 + 4 * q;
        const int px = X0 + lx, py = Y0 + ly;
        const bool in = px < W && py < H;
        dn[q] = !in;
        T[q] = 1;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            pre[q][c] = 0;
            C[q][c] = 0;
            gC[q][c] = 0;
        }
        if (in) {
            const int64_t p = (int64_t)py * W + px;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const R v = img[3 * p + c];
                const R diff = v - (R)gt[3 * p + c];
                C[q][c] = v;
                loss += fabs((double)diff);
                const R sg = diff > (R)0 ? (R)1 : (diff < (R)0 ? (R)-1 : (R)0);
                // dL/dC = sign(C - gt) / (H W 3)  (optim.py:124-125)
                gC[q][c] = sizeof(R) == 8 ? (R)((double)sg / npx3) : sg * (R)(1.0 / npx3);
            }
        }
    }

    for (uint32_t b0 = rg.x; b0 < stop; b0 += BWD_BATCH) {
        __syncthreads();
        const int nb = (int)min((uint32_t)BWD_BATCH, stop - b0);
        for (int k = threadIdx.x; k < nb; k += BWD_THREADS) {
            const uint32_t r = pvals[b0 + k];
            const SplatRec<R> rec = rrec[r];
            stage(sm[k], rmu[r], rec, X0, Y0);
            int tx0, tx1, ty0, ty1;
            win_tiles(rec.win, tx0, tx1, ty0, ty1);
            s_pidx[k] = roff[r] + (uint64_t)((ty - ty0) * (tx1 - tx0 + 1) + (tx - tx0));
        }
        __syncthreads();
        for (int k = 0; k < nb; ++k) {
            const Staged<R>& s = sm[k];
            R acc[9];
#pragma unroll
            for (int e = 0; e < 9; ++e) acc[e] = 0;
            bool any = false;
            const bool colin = lx >= s.wx0 && lx < s.wx1;
#pragma unroll
            for (int q = 0; q < BWD_PPT; ++q) {
                const int ly = ly0 + 4 * q;
                if (dn[q] || !colin || ly < s.wy0 || ly >= s.wy1) continue;
                any = true;
                R dx, dy;
                pixel_delta(s, lx, ly, X0, Y0, dx, dy);
                const R power = (R)-0.5 * (s.a * dx * dx + (R)2 * s.b * dx * dy + s.c * dy * dy);
                const R G = ss_exp<R>(power);
                const R oG = s.o * G;
                const R alpha = min(oG, (R)ALPHA_CAP);
                const R w = alpha * T[q];
                const R col[3] = {s.col0, s.col1, s.col2};
                const R inv1m = (R)1 / ((R)1 - alpha);
                R dal = 0;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    acc[c] += gC[q][c] * w;
                    const R S = C[q][c] - pre[q][c] - w * col[c];
                    dal += gC[q][c] * (col[c] * T[q] - S * inv1m);
                }
                if (oG < (R)ALPHA_CAP) {
                    acc[3] += dal * G;
                    const R gp = dal * alpha;
                    const R adx = s.a * dx + s.b * dy;
                    const R ady = s.b * dx + s.c * dy;
                    acc[4] += gp * adx;
                    acc[5] += gp * ady;
                    acc[6] += (R)0.5 * gp * adx * adx;
                    acc[7] += (R)0.5 * gp * adx * ady;
                    acc[8] += (R)0.5 * gp * ady * ady;
                }
#pragma unroll
                for (int c = 0; c < 3; ++c) pre[q][c] += w * col[c];
                T[q] = T[q] * ((R)1 - alpha);
                if (T[q] < (R)T_CUTOFF) dn[q] = true;
            }
            if (__any_sync(0xffffffffu, any)) {
                const R y = warp_reduce8<R>(acc, lane);
                const R z = warp_sum<R>(acc[8]);
                if ((lane & 3) == 0) s_red[warp][k][((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1)] = y;
                if (lane == 0) s_red[warp][k][8] = z;
            } else if (lane < 9) {
                s_red[warp][k][lane] = 0;
            }
        }
        __syncthreads();
        for (int e = threadIdx.x; e < nb * 9; e += BWD_THREADS) {
            const int k = e / 9, q = e % 9;
            R sum = 0;
#pragma unroll
            for (int w = 0; w < BWD_WARPS; ++w) sum += s_red[w][k][q];
            partials[s_pidx[k] * 9 + q] = sum;
        }
    }
    // pairs after every pixel of the tile saturated contribute nothing
    for (uint32_t i = stop + threadIdx.x; i < rg.y; i += BWD_THREADS) {
        const uint32_t r = pvals[i];
        const SplatRec<R> rec = rrec[r];
        int tx0, tx1, ty0, ty1;
        win_tiles(rec.win, tx0, tx1, ty0, ty1);
        const uint64_t p = roff[r] + (uint64_t)((ty - ty0) * (tx1 - tx0 + 1) + (tx - tx0));
#pragma unroll
        for (int q = 0; q < 9; ++q) partials[p * 9 + q] = 0;
    }
    loss = warp_sum<double>(loss);
    if (lane == 0) s_loss[warp] = loss;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int w = 0; w < BWD_WARPS; ++w) t += s_loss[w];
        tile_loss[tile] = t;
    }
}

__global__ void k_loss_reduce(const double* __restrict__ tile_loss, int n, double inv_npx, double* __restrict__ out) {
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
template <typename R>
__global__ void k_chain(ss_model m, ss_camera cam, ss_light L, const int64_t* __restrict__ subset,
                        const uint64_t* __restrict__ dkeys, const uint32_t* __restrict__ dvals,
                        const uint64_t* __restrict__ roff, const uint32_t* __restrict__ rcnt,
                        const R* __restrict__ partials, int64_t n_in, int cutoff, float* __restrict__ grad) {
    const int B = ss_sh_bases(m.sh_degree);
    const int64_t a = m.active_count;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_in; r += (int64_t)gridDim.x * blockDim.x) {
        if (dkeys[r] == ~0ull) continue;
        const int64_t j = dvals[r];
        const int64_t row = subset ? subset[j] : j;
        if (row >= a) continue;
        double g[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        const uint32_t cnt = rcnt[r];
        const R* pp = partials + roff[r] * 9;
        for (uint32_t i = 0; i < cnt; ++i)
#pragma unroll
            for (int e = 0; e < 9; ++e) g[e] += (double)pp[i * 9 + e];
        Proj P;
        ss_cam_point(cam, m.means + row * 3, P.d, P.mc);
        ss_project(cam, m.log_scales + row * 3, m.quaternions + row * 4, cutoff != 0, P);
        Shade S;
        const float* sh = m.sh_coeffs + row * 3 * B;
        ss_shade(L, m.log_scales + row * 3, sh, B, m.sh_degree, m.light_visibility[row], P.d, P.Rq, S);

        double gc[3];
        for (int c = 0; c < 3; ++c) gc[c] = (S.pre[c] > 0.0 && S.pre[c] < 1.0) ? g[c] : 0.0;
        const double go = g[3];
        const double gm[2] = {g[4], g[5]};
        const double G2[2][2] = {{g[6], g[7]}, {g[7], g[8]}};
        const double(&J)[2][3] = P.J;
        // gJ = (G2 + G2^T) J cov ; gV = J^T G2 J ; G3 = W^T gV W = R_cw gV R_cw^T
        double JC[2][3], JG[2][3];
        for (int l = 0; l < 3; ++l) {
            JC[0][l] = J[0][0] * P.cov[0][l] + J[0][2] * P.cov[2][l];
            JC[1][l] = J[1][1] * P.cov[1][l] + J[1][2] * P.cov[2][l];
        }
        double gJ[2][3];
        for (int aa = 0; aa < 2; ++aa)
            for (int l = 0; l < 3; ++l) gJ[aa][l] = 2.0 * (G2[aa][0] * JC[0][l] + G2[aa][1] * JC[1][l]);
        for (int aa = 0; aa < 2; ++aa)
            for (int l = 0; l < 3; ++l) JG[aa][l] = G2[aa][0] * J[0][l] + G2[aa][1] * J[1][l];
        double gV[3][3];
        for (int k = 0; k < 3; ++k)
            for (int l = 0; l < 3; ++l) gV[k][l] = J[0][k] * JG[0][l] + J[1][k] * JG[1][l];
        const double* Rc = cam.rot_cw;
        double tmp[3][3], G3[3][3];
        for (int i = 0; i < 3; ++i)
            for (int l = 0; l < 3; ++l)
                tmp[i][l] = Rc[i * 3 + 0] * gV[0][l] + Rc[i * 3 + 1] * gV[1][l] + Rc[i * 3 + 2] * gV[2][l];
        for (int i = 0; i < 3; ++i)
            for (int k = 0; k < 3; ++k)
                G3[i][k] = tmp[i][0] * Rc[k * 3 + 0] + tmp[i][1] * Rc[k * 3 + 1] + tmp[i][2] * Rc[k * 3 + 2];
        // mean path through mu2d and J
        const double x = P.mc[0], y = P.mc[1], z = P.mc[2];
        const double fx = cam.fx, fy = cam.fy, z2 = z * z, z3 = z2 * z;
        double gmc[3];
        gmc[0] = J[0][0] * gm[0] + gJ[0][2] * (-fx / z2);
        gmc[1] = J[1][1] * gm[1] + gJ[1][2] * (-fy / z2);
        gmc[2] = J[0][2] * gm[0] + J[1][2] * gm[1] + gJ[0][0] * (-fx / z2) + gJ[1][1] * (-fy / z2) +
                 gJ[0][2] * (2 * fx * x / z3) + gJ[1][2] * (2 * fy * y / z3);
        double gmean[3];
        for (int i = 0; i < 3; ++i) gmean[i] = Rc[i * 3 + 0] * gmc[0] + Rc[i * 3 + 1] * gmc[1] + Rc[i * 3 + 2] * gmc[2];
        // scales and rotation
        const double(&Rq)[3][3] = P.Rq;
        double gls[3];
        for (int k = 0; k < 3; ++k) {
            double t = 0;
            for (int b = 0; b < 3; ++b)
                for (int c = 0; c < 3; ++c) t += Rq[b][k] * G3[b][c] * Rq[c][k];
            gls[k] = t * 2.0 * P.S2[k];
        }
        double gR[3][3];
        for (int aa = 0; aa < 3; ++aa)
            for (int c = 0; c < 3; ++c) {
                double t = 0;
                for (int b = 0; b < 3; ++b) t += (G3[aa][b] + G3[b][aa]) * Rq[b][c];
                gR[aa][c] = t * P.S2[c];
            }
        double gcos = 0;
        for (int c = 0; c < 3; ++c) gcos += gc[c] * (S.albedo[c] * L.intensity[c]);
        gcos *= S.vis;
        const double gs = gcos * (S.s > 0 ? 1.0 : (S.s < 0 ? -1.0 : 0.0));
        for (int i = 0; i < 3; ++i) gR[i][S.axis] += gs * -L.direction[i];
        // quaternion through R(u), u = q/|q|
        const double w = P.u[0], qx = P.u[1], qy = P.u[2], qz = P.u[3];
        const double dR[4][3][3] = {
            {{0, -2 * qz, 2 * qy}, {2 * qz, 0, -2 * qx}, {-2 * qy, 2 * qx, 0}},
            {{0, 2 * qy, 2 * qz}, {2 * qy, -4 * qx, -2 * w}, {2 * qz, 2 * w, -4 * qx}},
            {{-4 * qy, 2 * qx, 2 * w}, {2 * qx, 0, 2 * qz}, {-2 * w, 2 * qz, -4 * qy}},
            {{-4 * qz, -2 * w, 2 * qx}, {2 * w, -4 * qz, 2 * qy}, {2 * qx, 2 * qy, 0}}};
        double h[4];
        for (int c = 0; c < 4; ++c) {
            double t = 0;
            for (int i = 0; i < 3; ++i)
                for (int jj = 0; jj < 3; ++jj) t += gR[i][jj] * dR[c][i][jj];
            h[c] = t;
        }
        double gq[4];
        const double udh = P.u[0] * h[0] + P.u[1] * h[1] + P.u[2] * h[2] + P.u[3] * h[3];
        for (int k = 0; k < 4; ++k) gq[k] = (h[k] - P.u[k] * udh) / P.qn;
        // appearance: SH coefficients
        const int64_t off_sh = 11 * a + row * 3 * B;
        const int BL = L.ambient_bands < B ? L.ambient_bands : B;
        for (int c = 0; c < 3; ++c) {
            for (int b = 0; b < B; ++b) {
                double v;
                if (L.ambient_bands == 0) v = gc[c] * S.Y[b];
                else v = (b < BL ? gc[c] * L.ambient[c * L.ambient_bands + b] : 0.0) + (b >= 1 ? gc[c] * S.Y[b] : 0.0);
                if (b == 0) v += gc[c] * (SS_SH_C0 * L.intensity[c]) * (S.cosv * S.vis);
                grad[off_sh + c * B + b] += (float)v;
            }
        }
        // view-direction path
        if (m.sh_degree > 0) {
            double dY[16][3];
            ss_sh_grad(S.vdir, m.sh_degree, dY);
            double gv[3] = {0, 0, 0};
            for (int c = 0; c < 3; ++c)
                for (int b = 1; b < B; ++b) {
                    const double t = sh[c * B + b] * gc[c];
                    gv[0] += t * dY[b][0];
                    gv[1] += t * dY[b][1];
                    gv[2] += t * dY[b][2];
                }
            const double vg = S.vdir[0] * gv[0] + S.vdir[1] * gv[1] + S.vdir[2] * gv[2];
            for (int i = 0; i < 3; ++i) gmean[i] += (gv[i] - S.vdir[i] * vg) / S.dist;
        }
        const double op = 1.0 / (1.0 + exp(-(double)m.logit_opacities[row]));
        for (int i = 0; i < 3; ++i) {
            grad[row * 3 + i] += (float)gmean[i];
            grad[3 * a + row * 3 + i] += (float)gls[i];
        }
        for (int k = 0; k < 4; ++k) grad[6 * a + row * 4 + k] += (float)gq[k];
        grad[10 * a + row] += (float)(go * op * (1.0 - op));
    }
}

// ---------------------------------------------------------------- host
inline int gridn(ss_ctx* ctx, int64_t n, int block = 256) {
    int64_t g = (n + block - 1) / block;
    int64_t cap = (int64_t)ctx->num_sms * 32;
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
    return SS_OK;
}

// K1..K4: preprocess, depth sort, count/scan/emit, tile sort, ranges.
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
    b.dkeys = SS_SCRATCH(ctx, uint64_t, na);
    b.dvals = SS_SCRATCH(ctx, uint32_t, na);
    uint64_t* kalt = SS_SCRATCH(ctx, uint64_t, na);
    uint32_t* valt = SS_SCRATCH(ctx, uint32_t, na);
    b.perg = SS_SCRATCH(ctx, PerG, na);
    b.rmu = SS_SCRATCH(ctx, double2, na);
    b.roff = SS_SCRATCH(ctx, uint64_t, na);
    b.rcnt = SS_SCRATCH(ctx, uint32_t, na);
    b.rrec = ss_scratch(ctx, sizeof(SplatRec<R>) * na);
    b.ranges = SS_SCRATCH(ctx, uint2, b.n_tiles);
    uint64_t* total = SS_SCRATCH(ctx, uint64_t, 1);
    if (!b.dkeys || !b.dvals || !kalt || !valt || !b.perg || !b.rmu || !b.roff || !b.rcnt || !b.rrec || !b.ranges ||
        !total)
        return SS_ERR_CUDA;
    SS_CUDA(ctx, cudaMemsetAsync(b.ranges, 0, sizeof(uint2) * b.n_tiles, s));
    DebugOut none;
    memset(&none, 0, sizeof(none));
    if (n > 0) {
        ss_tic(ctx, KC_PREPROCESS);
        k_preprocess<<<gridn(ctx, n, 128), 128, 0, s>>>(*m, *cam, *L, o->subset, n, o->extent_cutoff, b.dkeys, b.dvals,
                                                        b.perg, dbg ? *dbg : none);
        SS_CHECK_LAUNCH(ctx);
        ss_toc(ctx, KC_PREPROCESS);
        ss_tic(ctx, KC_DEPTH_SORT);
        SS_TRY(ss_radix_sort_u64(ctx, b.dkeys, b.dvals, kalt, valt, n, 64));
        ss_toc(ctx, KC_DEPTH_SORT);
        ss_tic(ctx, KC_BIN);
        k_count<R><<<gridn(ctx, n), 256, 0, s>>>(b.dkeys, b.dvals, b.perg, n, b.rmu, (SplatRec<R>*)b.rrec, b.rcnt);
        SS_CHECK_LAUNCH(ctx);
    } else {
        ss_tic(ctx, KC_BIN);
    }
    SS_TRY(ss_scan_u32_to_u64(ctx, b.rcnt, b.roff, n, total));
    ss_toc(ctx, KC_BIN);
    uint64_t P = 0;
    SS_TRY(ss_read_u64(ctx, total, &P));
    if (P > 0xffffffffull) return ss_fail(ctx, SS_ERR_CAPACITY, "too many tile overlaps (%llu)", (unsigned long long)P);
    b.pairs = (int64_t)P;
    const int64_t pa = P > 0 ? (int64_t)P : 1;
    b.pkeys = SS_SCRATCH(ctx, uint32_t, pa);
    b.pvals = SS_SCRATCH(ctx, uint32_t, pa);
    uint32_t* pk2 = SS_SCRATCH(ctx, uint32_t, pa);
    uint32_t* pv2 = SS_SCRATCH(ctx, uint32_t, pa);
    if (!b.pkeys || !b.pvals || !pk2 || !pv2) return SS_ERR_CUDA;
    if (P > 0) {
        ss_tic(ctx, KC_BIN);
        k_emit<R><<<gridn(ctx, n), 256, 0, s>>>((const SplatRec<R>*)b.rrec, b.rcnt, b.roff, n, b.tiles_x, b.pkeys,
                                                b.pvals);
        SS_CHECK_LAUNCH(ctx);
        ss_toc(ctx, KC_BIN);
        ss_tic(ctx, KC_TILE_SORT);
        SS_TRY(ss_radix_sort_u32(ctx, b.pkeys, b.pvals, pk2, pv2, (int64_t)P, b.tile_bits));
        ss_toc(ctx, KC_TILE_SORT);
        ss_tic(ctx, KC_BIN);
        k_ranges<<<gridn(ctx, (int64_t)P), 256, 0, s>>>(b.pkeys, (int64_t)P, b.ranges);
        SS_CHECK_LAUNCH(ctx);
        ss_toc(ctx, KC_BIN);
    }
    return SS_OK;
}

template <typename R>
int forward(ss_ctx* ctx, const ss_camera* cam, const ss_render_opts* o, const Bins& b, R* img, R* T,
            uint32_t* tile_stop) {
    ss_tic(ctx, KC_FORWARD);
    k_blend_fwd<R><<<b.n_tiles, FWD_THREADS, 0, ctx->stream>>>(
        b.ranges, b.pvals, b.rmu, (const SplatRec<R>*)b.rrec, cam->width, cam->height, b.tiles_x, o->background[0],
        o->background[1], o->background[2], img, T, tile_stop, ss_timing_on(ctx) ? ctx->dev_counters : nullptr);
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

template <typename R>
int backward_t(ss_ctx* ctx, const ss_model* m, const ss_camera* cam, const ss_light* L, const ss_render_opts* o,
               const float* gt, float* grad, double* loss, void* img_out, ss_render_stats* st) {
    cudaStream_t s = ctx->stream;
    Bins b;
    SS_TRY(build_bins<R>(ctx, m, cam, L, o, b, nullptr));
    const int64_t npx = (int64_t)cam->width * cam->height;
    R* img = img_out ? (R*)img_out : SS_SCRATCH(ctx, R, 3 * npx);
    uint32_t* stop = SS_SCRATCH(ctx, uint32_t, b.n_tiles);
    double* tloss = SS_SCRATCH(ctx, double, b.n_tiles);
    R* partials = SS_SCRATCH(ctx, R, 9 * (b.pairs > 0 ? b.pairs : 1));
    if (!img || !stop || !tloss || !partials) return SS_ERR_CUDA;
    SS_TRY(forward<R>(ctx, cam, o, b, img, (R*)nullptr, stop));
    const double inv_npx = 1.0 / (double)(3 * npx);
    ss_tic(ctx, KC_BACKWARD);
    k_blend_bwd<R><<<b.n_tiles, BWD_THREADS, 0, s>>>(b.ranges, b.pvals, b.rmu, (const SplatRec<R>*)b.rrec, b.roff, stop,
                                                      cam->width, cam->height, b.tiles_x, img, gt, (double)(3 * npx),
                                                      partials, tloss);
    SS_CHECK_LAUNCH(ctx);
    k_loss_reduce<<<1, 256, 0, s>>>(tloss, b.n_tiles, inv_npx, loss);
    SS_CHECK_LAUNCH(ctx);
    ss_toc(ctx, KC_BACKWARD);
    if (b.n_in > 0 && m->active_count > 0) {
        ss_tic(ctx, KC_CHAIN);
        k_chain<R><<<gridn(ctx, b.n_in, 128), 128, 0, s>>>(*m, *cam, *L, o->subset, b.dkeys, b.dvals, b.roff, b.rcnt,
                                                           partials, b.n_in, o->extent_cutoff, grad);
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

__global__ void k_order_out(const uint64_t* dkeys, const uint32_t* dvals, const uint64_t* vpos, int64_t n,
                            int64_t* order) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        if (dkeys[r] != ~0ull) order[r] = (int64_t)vpos[dvals[r]];
}

__global__ void k_debug_bins(const Bins b, int64_t* order_rows, const int64_t* subset, int64_t* ranges_out,
                             int64_t* pair_rank) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = tid; r < b.n_in; r += nt)
        if (order_rows && b.dkeys[r] != ~0ull) order_rows[r] = subset ? subset[b.dvals[r]] : (int64_t)b.dvals[r];
    for (int64_t t = tid; t < b.n_tiles; t += nt)
        if (ranges_out) {
            ranges_out[2 * t] = b.ranges[t].x;
            ranges_out[2 * t + 1] = b.ranges[t].y;
        }
    for (int64_t p = tid; p < b.pairs; p += nt)
        if (pair_rank) pair_rank[p] = b.pvals[p];
}

}  // namespace

extern "C" {

int ss_render(ss_ctx* ctx, const ss_model* m, const ss_camera* cam, const ss_light* L, const ss_render_opts* o,
              void* img, void* T, ss_render_stats* st) {
    if (!ctx) return SS_ERR_INVALID;
    SS_TRY(validate(ctx, m, cam, o));
    if (!img) return ss_fail(ctx, SS_ERR_INVALID, "image_out is required");
    SS_TRY(ss_scratch_reset(ctx));
    return o->precision ? render_t<double>(ctx, m, cam, L, o, img, T, st) : render_t<float>(ctx, m, cam, L, o, img, T, st);
}

int ss_backward(ss_ctx* ctx, const ss_model* m, const ss_camera* cam, const ss_light* L, const ss_render_opts* o,
                const float* gt, float* grad, double* loss, void* img, ss_render_stats* st) {
    if (!ctx) return SS_ERR_INVALID;
    SS_TRY(validate(ctx, m, cam, o));
    if (!gt || !grad || !loss) return ss_fail(ctx, SS_ERR_INVALID, "gt, grad_accum and loss_accum are required");
    SS_TRY(ss_scratch_reset(ctx));
    return o->precision ? backward_t<double>(ctx, m, cam, L, o, gt, grad, loss, img, st)
                        : backward_t<float>(ctx, m, cam, L, o, gt, grad, loss, img, st);
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
        k_visible_flags<<<gridn(ctx, n), 256, 0, s>>>(*m, *cam, o->subset, n, flag);
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
        k_order_out<<<gridn(ctx, n), 256, 0, s>>>(b.dkeys, b.dvals, vpos, n, out->order);
        SS_CHECK_LAUNCH(ctx);
    }
    if (visible_out) *visible_out = (int64_t)M;
    SS_CUDA(ctx, cudaStreamSynchronize(s));
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
    k_debug_bins<<<gridn(ctx, b.n_in > b.pairs ? b.n_in : b.pairs), 256, 0, ctx->stream>>>(b, order_rows, o->subset,
                                                                                          ranges_out, pair_rank);
    SS_CHECK_LAUNCH(ctx);
    if (st) {
        st->visible = -1;
        st->pairs = b.pairs;
        st->tiles = b.n_tiles;
    }
    SS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SS_OK;
}

}  // extern "C"
