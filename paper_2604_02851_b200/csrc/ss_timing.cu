// Per-kernel-class CUDA-event timing and the FP32 peak probe used by bench.py.
#include <vector>

#include "ss_internal.cuh"

namespace {
struct Span {
    int cls;
    cudaEvent_t a, b;
};
struct Timer {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    std::vector<Span> spans;
    cudaEvent_t open[KC_COUNT] = {};
    double ms[KC_COUNT] = {};
    int64_t groups[KC_COUNT] = {};
};
Timer* timer_of(const ss_ctx* c) { return (Timer*)c->timer_state; }

cudaEvent_t take(Timer* t) {
    if (!t->pool.empty()) {
        cudaEvent_t e = t->pool.back();
        t->pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

__global__ void k_fma_probe(float* out, int iters) {
    float a = threadIdx.x * 1e-3f, b = 0.999f, c0 = 1.0f, c1 = 0.5f, c2 = 0.25f, c3 = 0.125f;
    float x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = fmaf(x0, b, c0); x1 = fmaf(x1, b, c1); x2 = fmaf(x2, b, c2); x3 = fmaf(x3, b, c3);
        x4 = fmaf(x4, b, c0); x5 = fmaf(x5, b, c1); x6 = fmaf(x6, b, c2); x7 = fmaf(x7, b, c3);
    }
    float s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 12345.678f) out[0] = s;
}
}  // namespace

bool ss_timing_on(const ss_ctx* ctx) { return ctx->timer_state && timer_of(ctx)->on; }

void ss_tic(ss_ctx* ctx, int cls) {
    if (!ss_timing_on(ctx)) return;
    Timer* t = timer_of(ctx);
    cudaEvent_t e = take(t);
    cudaEventRecord(e, ctx->stream);
    t->open[cls] = e;
}

void ss_toc(ss_ctx* ctx, int cls) {
    if (!ss_timing_on(ctx)) return;
    Timer* t = timer_of(ctx);
    if (!t->open[cls]) return;
    cudaEvent_t e = take(t);
    cudaEventRecord(e, ctx->stream);
    t->spans.push_back({cls, t->open[cls], e});
    t->open[cls] = nullptr;
}

extern "C" {

int ss_set_timing(ss_ctx* ctx, int enable) {
    if (!ctx) return SS_ERR_INVALID;
    if (!ctx->timer_state) ctx->timer_state = new Timer();
    if (!ctx->dev_counters) {
        SS_CUDA(ctx, cudaMalloc(&ctx->dev_counters, 4 * sizeof(unsigned long long)));
        SS_CUDA(ctx, cudaMemsetAsync(ctx->dev_counters, 0, 4 * sizeof(unsigned long long), ctx->stream));
    }
    timer_of(ctx)->on = enable != 0;
    return SS_OK;
}

int ss_get_timing(ss_ctx* ctx, double ms_out[SS_KC_COUNT], int64_t groups_out[SS_KC_COUNT], uint64_t counters[4],
                  int reset) {
    if (!ctx || !ctx->timer_state) return SS_ERR_INVALID;
    Timer* t = timer_of(ctx);
    SS_CUDA(ctx, ss_stream_sync(ctx));
    for (auto& s : t->spans) {
        float ms = 0;
        cudaEventElapsedTime(&ms, s.a, s.b);
        t->ms[s.cls] += ms;
        t->groups[s.cls] += 1;
        t->pool.push_back(s.a);
        t->pool.push_back(s.b);
    }
    t->spans.clear();
    for (int i = 0; i < KC_COUNT; ++i) {
        if (ms_out) ms_out[i] = t->ms[i];
        if (groups_out) groups_out[i] = t->groups[i];
    }
    if (counters && ctx->dev_counters) {
        uint64_t tmp[4];
        SS_TRY(ss_read_u64(ctx, ctx->dev_counters, tmp, 4));
        for (int i = 0; i < 4; ++i) counters[i] = tmp[i];
        counters[1] = ctx->launches;  // host-side count of kernel launches
    }
    if (reset) {
        for (int i = 0; i < KC_COUNT; ++i) {
            t->ms[i] = 0;
            t->groups[i] = 0;
        }
        if (ctx->dev_counters) SS_CUDA(ctx, cudaMemsetAsync(ctx->dev_counters, 0, 4 * sizeof(unsigned long long), ctx->stream));
        ctx->launches = 0;
    }
    return SS_OK;
}

int ss_measure_fp32_peak(ss_ctx* ctx, double* tflops) {
    if (!ctx || !tflops) return SS_ERR_INVALID;
    float* out = nullptr;
    SS_CUDA(ctx, cudaMalloc(&out, 16));
    const int blocks = ctx->num_sms * 8, threads = 256, iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_fma_probe<<<blocks, threads, 0, ctx->stream>>>(out, 100);  // warm-up
    cudaEventRecord(a, ctx->stream);
    k_fma_probe<<<blocks, threads, 0, ctx->stream>>>(out, iters);
    cudaEventRecord(b, ctx->stream);
    SS_CUDA(ctx, cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    *tflops = 2.0 * 8.0 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
    return SS_OK;
}

}  // extern "C"
