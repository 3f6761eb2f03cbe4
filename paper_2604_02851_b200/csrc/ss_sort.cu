// Stable LSD radix sort of (key, uint32 value) pairs, 8-bit digits, one
// kernel per digit pass ("onesweep": Adinets & Merrill, 2022).
//
//   k_hist_all   one read of the keys -> global digit histograms of every pass
//   k_base_scan  exclusive scan of each pass's 256 counts -> digit base offsets
//   k_onesweep   per pass: a block takes the next 3072/4096-key tile (atomic tile
//                counter, so every earlier tile is already running), ranks its
//                keys stably with warp __match_any_sync, publishes its
//                per-digit counts, looks back over earlier tiles' published
//                counts/prefixes (decoupled look-back) to get its global digit
//                offsets, then writes each digit run coalesced from shared memory
//
// Per pass the keys and values are read once and written once.  Used for the
// depth sort of Gaussians (32-bit range-shifted keys, 4 passes) and the tile
// sort of (tile, splat) pairs (ceil(log2 tiles) bits, 2 passes at 1080p).
#include "ss_internal.cuh"

namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_MAX_PASSES = 8;
#ifndef RS_LB
#define RS_LB 8
#endif
constexpr int LB = RS_LB;  // look-back window (tiles per step)
#ifndef RS_MINB12
#define RS_MINB12 3  // blocks per SM asked of the 12-item (tile sort) and 16-item (depth sort) passes (measured)
#endif
#ifndef RS_MINB16
#define RS_MINB16 2
#endif
constexpr uint32_t FLAG_AGG = 1u << 30, FLAG_INC = 2u << 30, CNT_MASK = (1u << 30) - 1;

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename K>
__global__ void __launch_bounds__(RS_THREADS) k_hist_all(const K* __restrict__ keys, int64_t n, int key_bits,
                                                         uint32_t* __restrict__ hist, const uint64_t* __restrict__ n_dev) {
    SS_PDL_WAIT();
    if (n_dev) n = min(n, (int64_t)*n_dev);  // a device-side count (<= the launch capacity n)
    __shared__ uint32_t cnt[RS_MAX_PASSES][256];
    const int passes = (key_bits + 7) / 8;
    for (int p = 0; p < passes; ++p) cnt[p][threadIdx.x] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const K k = keys[i];
        for (int p = 0; p < passes; ++p) {
            const int bits = key_bits - 8 * p < 8 ? key_bits - 8 * p : 8;
            atomicAdd(&cnt[p][(unsigned)(k >> (8 * p)) & ((1u << bits) - 1u)], 1u);
        }
    }
    __syncthreads();
    for (int p = 0; p < passes; ++p)
        if (cnt[p][threadIdx.x]) atomicAdd(&hist[p * 256 + threadIdx.x], cnt[p][threadIdx.x]);
}

__global__ void k_base_scan(const uint32_t* __restrict__ hist, int passes, uint64_t* __restrict__ base) {
    SS_PDL_WAIT();
    // one warp per pass
    const int p = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (p >= passes) return;
    uint64_t run = 0;
    for (int c = 0; c < 256; c += 32) {
        const uint64_t v = hist[p * 256 + c + lane];
        uint64_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        base[p * 256 + c + lane] = run + incl - v;
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
}

template <typename K, int RS_ITEMS>
__global__ void __launch_bounds__(RS_THREADS, RS_ITEMS <= 12 ? RS_MINB12 : RS_MINB16) k_onesweep(const K* __restrict__ keys, const uint32_t* __restrict__ vals,
                                                         int64_t n, int shift, unsigned mask,
                                                         const uint64_t* __restrict__ digit_base,
                                                         uint32_t* __restrict__ part, unsigned* __restrict__ tile_ctr,
                                                         K* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                                                         const uint64_t* __restrict__ n_dev) {
    SS_PDL_WAIT();
    if (n_dev) n = min(n, (int64_t)*n_dev);  // a device-side count (<= the launch capacity n)
    constexpr int RS_TILE = RS_THREADS * RS_ITEMS;
    __shared__ K s_keys[RS_TILE];
    __shared__ uint32_t s_vals[RS_TILE];
    __shared__ uint32_t s_wcnt[RS_WARPS][256];
    __shared__ uint32_t s_run[256];
    __shared__ uint32_t s_start[256];
    __shared__ uint64_t s_goff[256];
    __shared__ uint32_t s_wsum[RS_WARPS];
    __shared__ unsigned s_tile;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
    s_run[tid] = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) s_wcnt[w][tid] = 0;
    __syncthreads();
    const unsigned tile = s_tile;
    const int64_t base = (int64_t)tile * RS_TILE;
    // tiles are taken in ticket order, so every tile past the (device-side)
    // count is preceded only by tiles that also leave: nobody waits on them
    if (base >= n && tile > 0) return;

    // ---- warp w owns keys [w*256, (w+1)*256) of the tile (item r at r*32 + lane):
    // load them all first, then rank within the warp without block barriers
    K k[RS_ITEMS];
    uint32_t v[RS_ITEMS];
    const int64_t wbase = base + (int64_t)warp * (RS_ITEMS * 32);
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        const bool ok = i < n;
        k[r] = ok ? keys[i] : K(0);
        v[r] = ok ? vals[i] : 0u;
    }
    uint32_t rank[RS_ITEMS];
    unsigned dig[RS_ITEMS];
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        const bool ok = i < n;
        const unsigned d = ok ? ((unsigned)(k[r] >> shift) & mask) : 256u + lane;  // invalid lanes match only themselves
        dig[r] = d;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const unsigned below = __popc(peers & lanemask_lt());
        const int leader = __ffs(peers) - 1;
        uint32_t prior = 0;
        if (ok && lane == leader) {
            prior = s_wcnt[warp][d];
            s_wcnt[warp][d] = prior + __popc(peers);
        }
        prior = __shfl_sync(0xffffffffu, prior, leader);
        rank[r] = prior + below;  // rank among the warp's keys of digit d
        __syncwarp();
    }
    __syncthreads();
    // per digit: offsets of each warp's run inside the tile's digit run, and the tile total
    {
        uint32_t acc = 0;
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) {
            const uint32_t c = s_wcnt[w][tid];
            s_wcnt[w][tid] = acc;
            acc += c;
        }
        s_run[tid] = acc;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r)
        if (dig[r] < 256u) rank[r] += s_wcnt[warp][dig[r]];

    // ---- decoupled look-back: this tile's global offset for digit `tid`
    {
        const uint32_t mine = s_run[tid];
        volatile uint32_t* slot = part + (int64_t)tile * 256 + tid;
        if (tile == 0) {
            *slot = FLAG_INC | mine;
            s_goff[tid] = digit_base[tid];
        } else {
            *slot = FLAG_AGG | mine;
            // look back LB tiles per step with independent loads (the chain of
            // dependent L2 round trips shrinks LB-fold); a window is used only
            // once every tile up to its nearest inclusive prefix has published
            uint64_t excl = 0;
            for (int64_t t = (int64_t)tile - 1; t >= 0;) {
                uint32_t w[LB];
#pragma unroll
                for (int k = 0; k < LB; ++k)
                    w[k] = t - k >= 0 ? *(const volatile uint32_t*)(part + (t - k) * 256 + tid) : (FLAG_INC | 0u);
                int stop = LB;
                bool ready = true;
#pragma unroll
                for (int k = LB - 1; k >= 0; --k) {
                    if ((w[k] & ~CNT_MASK) == 0) ready = false, stop = k;  // unpublished: must wait for it
                    else if (w[k] & FLAG_INC) ready = true, stop = k;
                }
                if (!ready) continue;
                uint64_t acc = 0;
#pragma unroll
                for (int k = 0; k < LB; ++k)
                    if (k <= stop) acc += w[k] & CNT_MASK;
                excl += acc;
                if (stop < LB) break;
                t -= LB;
            }
            *slot = FLAG_INC | (uint32_t)(excl + mine);
            s_goff[tid] = digit_base[tid] + excl;
        }
    }
    // exclusive scan of the tile's per-digit counts -> local run starts
    {
        const uint32_t c = s_run[tid];
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        uint32_t wpre = 0;
        for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
        s_start[tid] = wpre + incl - c;
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        if (dig[r] < 256u) {
            const uint32_t p = s_start[dig[r]] + rank[r];
            s_keys[p] = k[r];
            s_vals[p] = v[r];
        }
    }
    __syncthreads();
    const int64_t cnt = (n - base) < RS_TILE ? (n - base) : RS_TILE;
    for (int i = tid; i < cnt; i += RS_THREADS) {
        const K key = s_keys[i];
        const unsigned d = (unsigned)(key >> shift) & mask;
        const uint64_t o = s_goff[d] + (uint64_t)(i - s_start[d]);
        SS_ASSERT(o < (uint64_t)n);
        keys_out[o] = key;
        vals_out[o] = s_vals[i];
    }
}

template <typename K, int RS_ITEMS>
int sort_impl(ss_ctx* ctx, K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, int64_t n, int key_bits,
              const uint64_t* n_dev) {
    constexpr int RS_TILE = RS_THREADS * RS_ITEMS;
    if (n <= 1 || key_bits <= 0) return SS_OK;
    if (n > (int64_t)CNT_MASK) return ss_fail(ctx, SS_ERR_CAPACITY, "radix sort limited to 2^30 keys");
    const int passes = (key_bits + 7) / 8;
    const int64_t tiles = (n + RS_TILE - 1) / RS_TILE;
    uint32_t* hist = SS_SCRATCH(ctx, uint32_t, RS_MAX_PASSES * 256);
    uint64_t* base = SS_SCRATCH(ctx, uint64_t, RS_MAX_PASSES * 256);
    uint32_t* part = SS_SCRATCH(ctx, uint32_t, tiles * 256 * passes);
    unsigned* ctr = SS_SCRATCH(ctx, unsigned, RS_MAX_PASSES);
    if (!hist || !base || !part || !ctr) return SS_ERR_CUDA;
    cudaStream_t s = ctx->stream;
    SS_CUDA(ctx, cudaMemsetAsync(hist, 0, sizeof(uint32_t) * RS_MAX_PASSES * 256, s));
    SS_CUDA(ctx, cudaMemsetAsync(part, 0, sizeof(uint32_t) * tiles * 256 * passes, s));
    SS_CUDA(ctx, cudaMemsetAsync(ctr, 0, sizeof(unsigned) * RS_MAX_PASSES, s));
    int hb = (int)((n + RS_THREADS * 16 - 1) / (RS_THREADS * 16));
    if (hb > ctx->num_sms * 8) hb = ctx->num_sms * 8;
    SS_CUDA(ctx, ss_launch((k_hist_all<K>), dim3(hb), dim3(RS_THREADS), 0, s, keys, n, key_bits, hist, n_dev));
    SS_CHECK_LAUNCH(ctx);
    SS_CUDA(ctx, ss_launch((k_base_scan), dim3(1), dim3(32 * RS_MAX_PASSES), 0, s, hist, passes, base));
    SS_CHECK_LAUNCH(ctx);
    K* src_k = keys;
    uint32_t* src_v = vals;
    K* dst_k = keys_alt;
    uint32_t* dst_v = vals_alt;
    for (int p = 0; p < passes; ++p) {
        const int shift = 8 * p;
        const int bits = key_bits - shift < 8 ? key_bits - shift : 8;
        const unsigned mask = (1u << bits) - 1u;
        SS_CUDA(ctx, ss_launch((k_onesweep<K, RS_ITEMS>), dim3((unsigned)tiles), dim3(RS_THREADS), 0, s, src_k, src_v, n, shift, mask, base + p * 256,
                                                             part + (int64_t)p * tiles * 256, ctr + p, dst_k, dst_v, n_dev));
        SS_CHECK_LAUNCH(ctx);
        K* tk = src_k; src_k = dst_k; dst_k = tk;
        uint32_t* tv = src_v; src_v = dst_v; dst_v = tv;
    }
    if (src_k != keys) {
        SS_CUDA(ctx, cudaMemcpyAsync(keys, src_k, sizeof(K) * n, cudaMemcpyDeviceToDevice, s));
        SS_CUDA(ctx, cudaMemcpyAsync(vals, src_v, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s));
    }
    return SS_OK;
}

}  // namespace

int ss_radix_sort_u32(ss_ctx* ctx, uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                      int64_t n, int key_bits, const uint64_t* n_dev) {
    // tile size: 4096 keys for the 32-bit depth keys (fewer tiles, shorter
    // look-back chains), 3072 for the short tile-id keys of the (tile, splat)
    // pairs (measured: 2048 / 3072 / 4096 -> 1.17 / 1.11 / 1.22 ms per step)
#ifndef RS_SHORT_ITEMS
#define RS_SHORT_ITEMS 12
#endif
#ifndef RS_LONG_ITEMS
#define RS_LONG_ITEMS 16
#endif
    if (key_bits > 16) return sort_impl<uint32_t, RS_LONG_ITEMS>(ctx, keys, vals, keys_alt, vals_alt, n, key_bits, n_dev);
    return sort_impl<uint32_t, RS_SHORT_ITEMS>(ctx, keys, vals, keys_alt, vals_alt, n, key_bits, n_dev);
}
