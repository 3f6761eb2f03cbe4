// Context, error reporting, scratch arena and the host compression stage.
#include <stdarg.h>
#include <zlib.h>

#include <vector>

#include "ss_internal.cuh"

namespace {
struct Arena {
    std::vector<std::pair<uint8_t*, size_t>> blocks;  // (ptr, capacity)
    size_t used = 0;        // bytes used in the last block
    size_t call_total = 0;  // bytes requested since the last reset
    size_t high_water = 0;
};
Arena* arena_of(ss_ctx* c) { return (Arena*)c->arena_state; }
}  // namespace

int ss_fail(ss_ctx* ctx, int code, const char* fmt, ...) {
    if (ctx) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(ctx->err, sizeof(ctx->err), fmt, ap);
        va_end(ap);
    }
    return code;
}

int ss_scratch_reset(ss_ctx* ctx) {
    Arena* a = arena_of(ctx);
    if (a->call_total > a->high_water) a->high_water = a->call_total;
    if (a->blocks.size() > 1) {
        // coalesce into one block large enough for the biggest call seen
        SS_CUDA(ctx, ss_stream_sync(ctx));
        for (auto& b : a->blocks) cudaFree(b.first);
        a->blocks.clear();
        size_t cap = ss_align(a->high_water + a->high_water / 4 + (1 << 20));
        uint8_t* p = nullptr;
        SS_CUDA(ctx, cudaMalloc(&p, cap));
        a->blocks.push_back({p, cap});
    }
    a->used = 0;
    a->call_total = 0;
    return SS_OK;
}

void* ss_scratch(ss_ctx* ctx, size_t bytes) {
    Arena* a = arena_of(ctx);
    bytes = ss_align(bytes ? bytes : 1);
    a->call_total += bytes;
    if (a->blocks.empty() || a->used + bytes > a->blocks.back().second) {
        size_t cap = ss_align(bytes > (64u << 20) ? bytes : (64u << 20));
        uint8_t* p = nullptr;
        ++ctx->host_syncs;  // cudaMalloc may synchronise the device
        cudaError_t e = cudaMalloc(&p, cap);
        if (e != cudaSuccess) {
            ss_fail(ctx, SS_ERR_CUDA, "scratch cudaMalloc(%zu): %s", cap, cudaGetErrorString(e));
            return nullptr;
        }
        a->blocks.push_back({p, cap});
        a->used = 0;
    }
    void* out = a->blocks.back().first + a->used;
    a->used += bytes;
    return out;
}

int ss_read_u64(ss_ctx* ctx, const void* dev, uint64_t* out, int count) {
    SS_CUDA(ctx, cudaMemcpyAsync(ctx->pinned, dev, sizeof(uint64_t) * count, cudaMemcpyDeviceToHost, ctx->stream));
    SS_CUDA(ctx, ss_stream_sync(ctx));
    memcpy(out, ctx->pinned, sizeof(uint64_t) * count);
    return SS_OK;
}

extern "C" {

int ss_abi_version(void) { return SS_ABI_VERSION; }

int ss_ctx_create(int device, ss_ctx** out) {
    if (!out) return SS_ERR_INVALID;
    *out = nullptr;
    if (cudaSetDevice(device) != cudaSuccess) return SS_ERR_CUDA;
    ss_ctx* c = new ss_ctx();
    c->device = device;
    c->stream = 0;
    c->err[0] = 0;
    c->arena_state = new Arena();
    c->timer_state = nullptr;
    c->dev_counters = nullptr;
    c->launches = 0;
    c->stream_switch = nullptr;
    c->pair_cap = 0;
    c->host_syncs = 0;
    if (cudaMallocHost(&c->pinned, 4096) != cudaSuccess) {
        delete (Arena*)c->arena_state;
        delete c;
        return SS_ERR_CUDA;
    }
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    *out = c;
    return SS_OK;
}

void ss_ctx_destroy(ss_ctx* ctx) {
    if (!ctx) return;
    ss_stream_sync(ctx);
    Arena* a = arena_of(ctx);
    for (auto& b : a->blocks) cudaFree(b.first);
    delete a;
    cudaFreeHost(ctx->pinned);
    if (ctx->dev_counters) cudaFree(ctx->dev_counters);
    if (ctx->stream_switch) cudaEventDestroy(ctx->stream_switch);
    // timer events are released with the context's device state
    delete ctx;
}

const char* ss_last_error(const ss_ctx* ctx) { return ctx ? ctx->err : "null context"; }

int64_t ss_host_syncs(const ss_ctx* ctx) { return ctx ? ctx->host_syncs : -1; }

int64_t ss_pair_capacity(ss_ctx* ctx, int64_t cap) {
    if (!ctx) return -1;
    if (cap > ctx->pair_cap) ctx->pair_cap = cap;
    else if (cap < 0) ctx->pair_cap = -cap;  // tests: force a (small) capacity to exercise the overflow path
    return ctx->pair_cap;
}

int ss_set_stream(ss_ctx* ctx, void* stream) {
    if (!ctx) return SS_ERR_INVALID;
    cudaStream_t next = (cudaStream_t)stream;
    if (next != ctx->stream) {
        // work already queued on the old stream may still read or write the
        // scratch arena the next call reuses: the new stream waits for it
        if (!ctx->stream_switch)
            SS_CUDA(ctx, cudaEventCreateWithFlags(&ctx->stream_switch, cudaEventDisableTiming));
        SS_CUDA(ctx, cudaEventRecord(ctx->stream_switch, ctx->stream));
        SS_CUDA(ctx, cudaStreamWaitEvent(next, ctx->stream_switch, 0));
        ctx->stream = next;
    }
    return SS_OK;
}

int64_t ss_grad_layout(int64_t a, int32_t sh_degree, int64_t off[5]) {
    int64_t B = (int64_t)(sh_degree + 1) * (sh_degree + 1);
    if (off) {
        off[0] = 0;
        off[1] = 3 * a;
        off[2] = 6 * a;
        off[3] = 10 * a;
        off[4] = 11 * a;
    }
    return a * (11 + 3 * B);
}

uint64_t ss_host_zlib_bound(uint64_t n) { return (uint64_t)compressBound((uLong)n); }

int ss_host_zlib_compress(const uint8_t* src, uint64_t n, uint8_t* dst, uint64_t cap, uint64_t* out_len) {
    uLongf dl = (uLongf)cap;
    // compress2(level 6) == Python zlib.compress(data, level=6): same
    // deflateInit defaults (window 15, memLevel 8, default strategy)
    int rc = compress2(dst, &dl, src, (uLong)n, 6);
    if (rc != Z_OK) return SS_ERR_CAPACITY;
    *out_len = dl;
    return SS_OK;
}

}  // extern "C"
