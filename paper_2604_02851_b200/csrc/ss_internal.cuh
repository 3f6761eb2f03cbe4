// Internal definitions shared by the sm_100a translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/splatstream_b200.h"
#include <nvtx3/nvToolsExt.h>

// An NVTX range over a public entry point (visible in Nsight Systems / ncu
// range filters): SS_NVTX("ss_backward");
struct SsNvtxRange {
    explicit SsNvtxRange(const char* name) { nvtxRangePushA(name); }
    ~SsNvtxRange() { nvtxRangePop(); }
};
#define SS_NVTX(name) SsNvtxRange _ss_nvtx_range(name)

struct ss_ctx {
    int device;
    cudaStream_t stream;
    char err[512];
    // grow-only device scratch arena (see ss_ctx.cu): one block in steady
    // state; a call that outgrows it spills into extra blocks, which are
    // coalesced into one larger block at the next reset
    void* arena_state;
    // small pinned host buffer for scalar read-backs
    void* pinned;
    int num_sms;
    // optional per-kernel-class CUDA-event timing (ss_set_timing)
    void* timer_state;
    unsigned long long* dev_counters;  // [0] T-gated (pixel, splat) evaluations
    unsigned long long launches;       // kernels launched through this context
    // orders a new stream after the previous one when ss_set_stream switches
    // (the scratch arena is shared by every call on the ctx)
    cudaEvent_t stream_switch;
    // pair capacity of sync-free binning (grow-only; 0 = unknown: the next
    // binning reads its pair count back once and sets it)
    int64_t pair_cap;
    // host synchronisations the library issued (stream syncs, read-backs,
    // scratch-arena allocations): ss_host_syncs, for the sync-free tests
    int64_t host_syncs;
};

enum ss_kernel_class {
    KC_PREPROCESS = 0, KC_DEPTH_SORT, KC_BIN, KC_TILE_SORT, KC_FORWARD, KC_BACKWARD, KC_CHAIN, KC_ADAM, KC_CODEC,
    KC_COUNT
};
// Bracket the launches of one kernel class with events on the ctx stream
// (no-ops unless timing is enabled).
void ss_tic(ss_ctx* ctx, int cls);
void ss_toc(ss_ctx* ctx, int cls);
bool ss_timing_on(const ss_ctx* ctx);

// ---------------------------------------------------------------- errors
int ss_fail(ss_ctx* ctx, int code, const char* fmt, ...);

#define SS_CUDA(ctx, expr)                                                              \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            return ss_fail((ctx), SS_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr, \
                           cudaGetErrorString(_e));                                     \
    } while (0)

// every kernel launch site is followed by SS_CHECK_LAUNCH, which also counts it
// Programmatic dependent launch (sm_90+): a kernel launched with ss_launch
// may be scheduled while its predecessor on the stream is still finishing;
// it waits at SS_PDL_WAIT() (its first statement) until the predecessor's
// results are visible, so the launch latency overlaps the predecessor's tail.
#define SS_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")

template <typename... KArgs, typename... Args>
inline cudaError_t ss_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                             Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Device-side invariants of the checked build (-DSS_CHECKS): a violated
// index bound traps the kernel (the launch then fails loudly).  compute-
// sanitizer is closed on the GPU pool, so this build is the bounds checker.
#ifdef SS_CHECKS
#define SS_ASSERT(cond)          \
    do {                         \
        if (!(cond)) __trap();   \
    } while (0)
#else
#define SS_ASSERT(cond) \
    do {                \
    } while (0)
#endif

#define SS_CHECK_LAUNCH(ctx)           \
    do {                               \
        ++(ctx)->launches;             \
        SS_CUDA(ctx, cudaGetLastError()); \
    } while (0)

#define SS_TRY(expr)            \
    do {                        \
        int _rc = (expr);       \
        if (_rc != SS_OK)       \
            return _rc;         \
    } while (0)

// ---------------------------------------------------------------- scratch
// Reset at the start of each public call; pointers are 256-byte aligned and
// stay valid until the next reset.  ss_scratch returns NULL (and sets the
// error) only if cudaMalloc fails.
int ss_scratch_reset(ss_ctx* ctx);
void* ss_scratch(ss_ctx* ctx, size_t bytes);
#define SS_SCRATCH(ctx, T, n) ((T*)ss_scratch((ctx), sizeof(T) * (size_t)(n)))
inline size_t ss_align(size_t b) { return (b + 255) & ~size_t(255); }

// peer replicas a fused parameter update can store into (ss_adam_step_peers)
#define SS_MAX_PEERS 15

// every host synchronisation of the library goes through here (counted)
inline cudaError_t ss_stream_sync(ss_ctx* ctx) {
    ++ctx->host_syncs;
    return cudaStreamSynchronize(ctx->stream);
}
// read a device scalar back to the host (synchronises the ctx stream)
int ss_read_u64(ss_ctx* ctx, const void* dev, uint64_t* out, int count = 1);

// ---------------------------------------------------------------- device math
// IEEE-exact double ops that nvcc never contracts into FMAs.  The fp64
// preprocess (windows, depth), the quantizers and Adam use these so the
// results equal the CPU oracle / reference numpy bit for bit.
__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dd(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsq(double a) { return __dsqrt_rn(a); }

// Deterministic exp from IEEE-exact ops (mirrors oracle/raster.py det_exp).
__device__ __forceinline__ double ss_det_exp(double x) {
    const double LN2_HI = 6.93147180369123816490e-01;
    const double LN2_LO = 1.90821492927058770002e-10;
    const double INV_LN2 = 1.44269504088896338700e+00;
    double k = rint(dm(x, INV_LN2));
    double r = ds(ds(x, dm(k, LN2_HI)), dm(k, LN2_LO));
    // 1/k! for k = 0..13, as the oracle computes them
    const double c[14] = {1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664,
                          0.008333333333333333, 0.001388888888888889, 0.0001984126984126984,
                          2.48015873015873e-05, 2.7557319223985893e-06, 2.755731922398589e-07,
                          2.505210838544172e-08, 2.08767569878681e-09, 1.6059043836821613e-10};
    double p = c[13];
#pragma unroll
    for (int i = 12; i >= 0; --i) p = da(dm(p, r), c[i]);
    return scalbn(p, (int)k);
}

// ---------------------------------------------------------------- scan / sort
// Exclusive scan of n uint32 values into uint64 (out may alias nothing);
// *total (device, may be NULL) receives the sum.
int ss_scan_u32_to_u64(ss_ctx* ctx, const uint32_t* in, uint64_t* out, int64_t n, uint64_t* total);
int ss_scan_u8_to_u64(ss_ctx* ctx, const uint8_t* in, uint64_t* out, int64_t n, uint64_t* total);
// Stable LSD radix sort of (key, value) pairs on bits [0, key_bits).
// keys/vals are sorted in place; alt buffers are scratch of the same size.
// With n_dev (device), the first *n_dev <= n entries are sorted (n sizes the
// launch: no host read of the count).
int ss_radix_sort_u32(ss_ctx* ctx, uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                      int64_t n, int key_bits, const uint64_t* n_dev = nullptr);

inline int ss_grid(int64_t n, int block) { return (int)((n + block - 1) / block); }
