// CRC-32 of the frame envelope (ref protocol/framing.py:51-53: zlib.crc32
// over header + payload), computed where the payload already is: in HBM.
//
// CRC-32 (reflected polynomial 0xEDB88320, init/xorout 0xFFFFFFFF) is affine
// over GF(2): with S(s, M) the register after feeding M from state s,
//   S(s, M) = s * x^(8|M|) mod P  xor  S(0, M)
// and S(0, .) ignores leading zero bytes.  So the message is cut into
// SEG-byte segments counted from its END (the first segment is the short one,
// implicitly zero-padded in front); thread t of block b owns segment
// e = b*256 + t and contributes S(0, seg) * x^(8 * e * SEG).  Contributions
// XOR together (order-free, so the atomic combine is deterministic), and
// block 0 adds the init term ~0 * x^(8n) ^ ~0.  The factor is applied in two
// steps: x^(8 t SEG) by each thread, then x^(8 * 256 b SEG) to the block's
// XOR by one thread; the powers come from host-built digit tables (XTab).
// Segment remainders use a slice-by-4 table in shared memory.
//
// ss_crc32_combine is the host-side counterpart (zlib's crc32_combine
// semantics) used to prepend the frame header's CRC.
#include "ss_internal.cuh"

namespace {

constexpr uint32_t CRC_POLY = 0xEDB88320u;
constexpr int CRC_THREADS = 256;
constexpr int CRC_SEG = 256;  // bytes per thread (a multiple of 16)

struct X2N {
    uint32_t v[64];  // x^(2^k) mod P, reflected
};

// x^(8 m) for the offsets the kernel needs, by digits of m (SEG = 256):
//   A[i] = x^(8 i), B[i] = x^(8 * 256 i)  (i < 256; B is the per-thread factor)
//   C[i] = x^(8 * 65536 i), D[i] = x^(8 * 2^22 i)  (i < 64)
// so any m < 2^28 (the payload cap) costs at most 4 multiplications
constexpr int CRC_TAB = 256 + 256 + 64 + 64;
struct XTab {
    uint32_t v[CRC_TAB];
};

// a * b mod P (reflected: bit 31 is x^0)
__host__ __device__ inline uint32_t gf_mul(uint32_t a, uint32_t b) {
    uint32_t p = 0;
#pragma unroll 4
    for (int i = 0; i < 32; ++i) {
        p ^= b & (0u - ((a >> (31 - i)) & 1u));
        b = (b >> 1) ^ (CRC_POLY & (0u - (b & 1u)));
    }
    return p;
}

// x^(8 n) mod P from the x^(2^k) table
__host__ __device__ inline uint32_t x8n(uint64_t n, const uint32_t* x2n) {
    uint32_t p = 0x80000000u;  // x^0
    int k = 3;
    while (n) {
        if (n & 1) p = gf_mul(x2n[k & 63], p);
        n >>= 1;
        ++k;
    }
    return p;
}

// x^(8 m) mod P from the digit tables (m < 2^28), else the x^(2^k) loop
__device__ __forceinline__ uint32_t x8m_tab(uint64_t m, const uint32_t* tab, const uint32_t* x2n) {
    if (m >> 28) return x8n(m, x2n);
    uint32_t p = tab[m & 255];
    if ((m >> 8) & 255) p = gf_mul(tab[256 + ((m >> 8) & 255)], p);
    if ((m >> 16) & 63) p = gf_mul(tab[512 + ((m >> 16) & 63)], p);
    if (m >> 22) p = gf_mul(tab[576 + (m >> 22)], p);
    return p;
}

X2N make_x2n() {
    X2N t;
    uint32_t p = 0x40000000u;  // x^1
    for (int k = 0; k < 64; ++k) {
        t.v[k] = p;
        p = gf_mul(p, p);
    }
    return t;
}

__device__ __forceinline__ uint32_t crc_byte(uint32_t s, uint32_t b, const uint32_t* T0) {
    return T0[(s ^ b) & 0xffu] ^ (s >> 8);
}

__device__ __forceinline__ uint32_t crc_word(uint32_t s, uint32_t w, const uint32_t (*T)[256]) {
    s ^= w;
    return T[3][s & 0xffu] ^ T[2][(s >> 8) & 0xffu] ^ T[1][(s >> 16) & 0xffu] ^ T[0][s >> 24];
}

__global__ void __launch_bounds__(CRC_THREADS) k_crc32(const uint8_t* __restrict__ data, const uint64_t* __restrict__ len_dev,
                                                       uint64_t len, uint32_t* __restrict__ out, X2N x2n, XTab xt) {
    SS_PDL_WAIT();
    const uint64_t n = len_dev ? min(*len_dev, len) : len;  // grids are sized for the bound
    if (blockIdx.x && (uint64_t)blockIdx.x * CRC_THREADS * CRC_SEG >= n) return;
    __shared__ uint32_t T[4][256];
    __shared__ uint32_t s_x2n[64];
    __shared__ uint32_t s_acc[CRC_THREADS / 32];
    __shared__ uint32_t s_tab[CRC_TAB];
    const int t = threadIdx.x;
    for (int i = t; i < CRC_TAB; i += CRC_THREADS) s_tab[i] = xt.v[i];
    {
        uint32_t c = (uint32_t)t;
#pragma unroll
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (CRC_POLY & (0u - (c & 1u)));
        T[0][t] = c;
        if (t < 64) s_x2n[t] = x2n.v[t];
    }
    __syncthreads();
#pragma unroll
    for (int j = 1; j < 4; ++j) {
        const uint32_t p = T[j - 1][t];
        T[j][t] = (p >> 8) ^ T[0][p & 0xffu];
        __syncthreads();
    }
    const uint64_t e = (uint64_t)blockIdx.x * CRC_THREADS + t;  // segment index from the end
    uint32_t contrib = 0;
    if (e * CRC_SEG < n) {
        const uint64_t end = n - e * CRC_SEG;
        const uint64_t beg = end > CRC_SEG ? end - CRC_SEG : 0;
        uint32_t s = 0;
        uint64_t i = beg;
        const uint64_t a0 = min(beg + ((16 - ((uintptr_t)(data + beg) & 15)) & 15), end);  // 16-byte aligned body
        for (; i < a0; ++i) s = crc_byte(s, data[i], T[0]);
        for (; i + 16 <= end; i += 16) {
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(data + i));
            s = crc_word(s, v.x, T);
            s = crc_word(s, v.y, T);
            s = crc_word(s, v.z, T);
            s = crc_word(s, v.w, T);
        }
        for (; i < end; ++i) s = crc_byte(s, data[i], T[0]);
        contrib = gf_mul(s_tab[256 + t], s);  // x^(8 * 256 t)
    }
    contrib = __reduce_xor_sync(0xffffffffu, contrib);
    if ((t & 31) == 0) s_acc[t >> 5] = contrib;
    __syncthreads();
    if (t == 0) {
        uint32_t b = 0;
#pragma unroll
        for (int w = 0; w < CRC_THREADS / 32; ++w) b ^= s_acc[w];
        if (b) b = gf_mul(x8m_tab((uint64_t)blockIdx.x * CRC_THREADS * CRC_SEG, s_tab, s_x2n), b);
        if (blockIdx.x == 0) b ^= gf_mul(x8m_tab(n, s_tab, s_x2n), 0xffffffffu) ^ 0xffffffffu;  // init / xorout
        if (b) atomicXor(out, b);
    }
}

const X2N& x2n_table() {
    static const X2N t = make_x2n();
    return t;
}

XTab make_xtab() {
    XTab t;
    const uint32_t* x2n = x2n_table().v;
    for (int i = 0; i < 256; ++i) {
        t.v[i] = x8n((uint64_t)i, x2n);
        t.v[256 + i] = x8n((uint64_t)i << 8, x2n);
    }
    for (int i = 0; i < 64; ++i) {
        t.v[512 + i] = x8n((uint64_t)i << 16, x2n);
        t.v[576 + i] = x8n((uint64_t)i << 22, x2n);
    }
    return t;
}

const XTab& xtab() {
    static const XTab t = make_xtab();
    return t;
}

}  // namespace

extern "C" int ss_crc32(ss_ctx* ctx, const uint8_t* data, const uint64_t* len_dev, uint64_t len, uint32_t* crc_out) {
    if (!ctx || !crc_out || (!data && len)) return SS_ERR_INVALID;
    SS_CUDA(ctx, cudaMemsetAsync(crc_out, 0, sizeof(uint32_t), ctx->stream));
    const uint64_t segs = (len + CRC_SEG - 1) / CRC_SEG;
    const uint64_t blocks = segs ? (segs + CRC_THREADS - 1) / CRC_THREADS : 1;
    if (blocks > 0x7fffffffull) return ss_fail(ctx, SS_ERR_INVALID, "crc32 input too large");
    ss_tic(ctx, KC_CODEC);
    SS_CUDA(ctx, ss_launch((k_crc32), dim3((unsigned)blocks), dim3(CRC_THREADS), 0, ctx->stream, data, len_dev, len, crc_out,
                           x2n_table(), xtab()));
    SS_CHECK_LAUNCH(ctx);
    ss_toc(ctx, KC_CODEC);
    return SS_OK;
}

extern "C" uint32_t ss_crc32_combine(uint32_t crc1, uint32_t crc2, uint64_t len2) {
    return gf_mul(x8n(len2, x2n_table().v), crc1) ^ crc2;
}
