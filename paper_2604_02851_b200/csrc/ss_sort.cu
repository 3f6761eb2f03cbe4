// Stable LSD radix sort of (key, uint32 value) pairs, 8-bit digits.
//
// Per pass: (1) upsweep -- per-block digit histogram (digit-major so one scan
// yields every block's global offset per digit); (2) exclusive scan of the
// histogram; (3) downsweep -- stable in-block ranking with warp
// __match_any_sync, local scatter into shared memory in digit order, then a
// coalesced write of each digit run to its global offset.
//
// Used twice per view: the depth sort of Gaussians (64-bit fp64-depth keys,
// exact reference order) and the tile sort of (tile, splat) pairs (only
// ceil(log2 tiles) key bits).
#include "ss_internal.cuh"

namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 8;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;
constexpr int RS_WARPS = RS_THREADS / 32;

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename K>
__global__ void __launch_bounds__(RS_THREADS) k_upsweep(const K* __restrict__ keys, int64_t n, int shift,
                                                        unsigned mask, int nb, uint32_t* __restrict__ hist) {
    __shared__ uint32_t cnt[256];
    cnt[threadIdx.x] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        int64_t i = base + r * RS_THREADS + threadIdx.x;
        if (i < n) atomicAdd(&cnt[(unsigned)(keys[i] >> shift) & mask], 1u);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * nb + blockIdx.x] = cnt[threadIdx.x];
}

template <typename K>
__global__ void __launch_bounds__(RS_THREADS) k_downsweep(const K* __restrict__ keys, const uint32_t* __restrict__ vals,
                                                          int64_t n, int shift, unsigned mask, int nb,
                                                          const uint64_t* __restrict__ offsets,
                                                          K* __restrict__ keys_out, uint32_t* __restrict__ vals_out) {
    __shared__ K s_keys[RS_TILE];
    __shared__ uint32_t s_vals[RS_TILE];
    __shared__ uint32_t s_wcnt[RS_WARPS][256];
    __shared__ uint32_t s_run[256];
    __shared__ uint32_t s_start[256];
    __shared__ uint64_t s_goff[256];
    __shared__ uint32_t s_wsum[RS_WARPS];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    s_run[tid] = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) s_wcnt[w][tid] = 0;
    s_goff[tid] = offsets[(int64_t)tid * nb + blockIdx.x];
    __syncthreads();

    K k[RS_ITEMS];
    uint32_t v[RS_ITEMS];
    uint32_t rank[RS_ITEMS];
    unsigned dig[RS_ITEMS];
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        int64_t i = base + r * RS_THREADS + tid;
        bool ok = i < n;
        k[r] = ok ? keys[i] : K(0);
        v[r] = ok ? vals[i] : 0u;
        unsigned d = ok ? ((unsigned)(k[r] >> shift) & mask) : 256u + lane;  // invalid lanes match only themselves
        dig[r] = d;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        unsigned below = __popc(peers & lanemask_lt());
        if (ok && below == 0) s_wcnt[warp][d] = __popc(peers);
        __syncthreads();
        if (ok) {
            uint32_t pre = s_run[d];
            for (int w = 0; w < warp; ++w) pre += s_wcnt[w][d];
            rank[r] = pre + below;
        }
        __syncthreads();
        uint32_t add = 0;
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) {
            add += s_wcnt[w][tid];
            s_wcnt[w][tid] = 0;
        }
        s_run[tid] += add;
        __syncthreads();
    }
    // exclusive scan of the block's per-digit totals -> local run starts
    {
        uint32_t c = s_run[tid];
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
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
            uint32_t p = s_start[dig[r]] + rank[r];
            s_keys[p] = k[r];
            s_vals[p] = v[r];
        }
    }
    __syncthreads();
    const int64_t cnt = (n - base) < RS_TILE ? (n - base) : RS_TILE;
    for (int i = tid; i < cnt; i += RS_THREADS) {
        K key = s_keys[i];
        unsigned d = (unsigned)(key >> shift) & mask;
        uint64_t o = s_goff[d] + (uint64_t)(i - s_start[d]);
        keys_out[o] = key;
        vals_out[o] = s_vals[i];
    }
}

template <typename K>
int sort_impl(ss_ctx* ctx, K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, int64_t n, int key_bits) {
    if (n <= 1 || key_bits <= 0) return SS_OK;
    const int nb = (int)((n + RS_TILE - 1) / RS_TILE);
    uint32_t* hist = SS_SCRATCH(ctx, uint32_t, (int64_t)256 * nb);
    uint64_t* offs = SS_SCRATCH(ctx, uint64_t, (int64_t)256 * nb);
    if (!hist || !offs) return SS_ERR_CUDA;
    K* src_k = keys;
    uint32_t* src_v = vals;
    K* dst_k = keys_alt;
    uint32_t* dst_v = vals_alt;
    for (int shift = 0; shift < key_bits; shift += 8) {
        int bits = key_bits - shift < 8 ? key_bits - shift : 8;
        unsigned mask = (1u << bits) - 1u;
        k_upsweep<K><<<nb, RS_THREADS, 0, ctx->stream>>>(src_k, n, shift, mask, nb, hist);
        SS_CHECK_LAUNCH(ctx);
        SS_TRY(ss_scan_u32_to_u64(ctx, hist, offs, (int64_t)256 * nb, nullptr));
        k_downsweep<K><<<nb, RS_THREADS, 0, ctx->stream>>>(src_k, src_v, n, shift, mask, nb, offs, dst_k, dst_v);
        SS_CHECK_LAUNCH(ctx);
        K* tk = src_k; src_k = dst_k; dst_k = tk;
        uint32_t* tv = src_v; src_v = dst_v; dst_v = tv;
    }
    if (src_k != keys) {
        SS_CUDA(ctx, cudaMemcpyAsync(keys, src_k, sizeof(K) * n, cudaMemcpyDeviceToDevice, ctx->stream));
        SS_CUDA(ctx, cudaMemcpyAsync(vals, src_v, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    return SS_OK;
}

}  // namespace

int ss_radix_sort_u64(ss_ctx* ctx, uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt,
                      int64_t n, int key_bits) {
    return sort_impl<uint64_t>(ctx, keys, vals, keys_alt, vals_alt, n, key_bits);
}

int ss_radix_sort_u32(ss_ctx* ctx, uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                      int64_t n, int key_bits) {
    return sort_impl<uint32_t>(ctx, keys, vals, keys_alt, vals_alt, n, key_bits);
}
