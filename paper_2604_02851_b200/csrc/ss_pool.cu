// Pool maintenance on the GPU: the per-tick row
// bookkeeping of the server, exact with the reference.
//
//   ss_select_rows     row predicates -> ascending int64 row indices (flag +
//                      exclusive scan + scatter):
//                        freeze_policy   ref expansion.py:134-142
//                        prune           ref expansion.py:184-197 (fp64 sigmoid)
//                        precull         ref expansion.py:145-181 (cell-centre
//                                        frustum / depth test per camera)
//   ss_gather_rows     new_row[i] = old_row[map[i]] over every column, with
//                      map[i] < 0 selecting a placeholder row (ref
//                      model.py:153-165 permute / remove_rows, model.py:327
//                      placeholder_batch for client-side appends)
//   ss_grid_rebuild    GridIndex.rebuild (ref model.py:418-426): cell of every
//                      row, a stable sort by cell, cells in first-appearance
//                      order (the dict order) with their member rows
//   ss_zigzag_varints  the permutation block of an ordering packet before
//                      its zlib stage (ref protocol/packets.py:153-158)
#include "ss_internal.cuh"

namespace {

inline int grid_for(ss_ctx* ctx, int64_t n) {
    const int64_t g = (n + 255) / 256;
    const int64_t cap = (int64_t)ctx->num_sms * 16;
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// camera-space point, (p - pos) @ R in the oracle's op order
__device__ __forceinline__ void cam_point(const ss_pool_camera& c, const double p[3], double out[3]) {
    const double d[3] = {ds(p[0], c.position[0]), ds(p[1], c.position[1]), ds(p[2], c.position[2])};
#pragma unroll
    for (int j = 0; j < 3; ++j)
        out[j] = da(da(dm(d[0], c.rot_cw[0 * 3 + j]), dm(d[1], c.rot_cw[1 * 3 + j])), dm(d[2], c.rot_cw[2 * 3 + j]));
}

// floor((p - origin) / cell) per axis (GridIndex.cells_of, model.py:406-407)
__device__ __forceinline__ void cell_of(const float* p, const double origin[3], double cell, int64_t c[3]) {
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = (int64_t)floor(dd(ds((double)p[k], origin[k]), cell));
}

__global__ void k_select_flags(ss_select s, uint8_t* __restrict__ flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += (int64_t)gridDim.x * blockDim.x) {
        bool keep = false;
        if (s.kind == SS_SELECT_FREEZE) {
            keep = s.age[i] >= s.age_threshold && s.grad_ema[i] < s.grad_threshold;  // expansion.py:140-141
        } else if (s.kind == SS_SELECT_PRUNE) {
            const double op = dd(1.0, da(1.0, exp(-(double)s.logits[i])));  // expansion.py:193
            keep = op < s.opacity_floor;
        } else {  // precull: the row's cell centre against every camera (expansion.py:160-180)
            const int64_t* ck = s.cells + 3 * i;
            double ctr[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) ctr[k] = da(s.origin[k], dm(da((double)ck[k], 0.5), s.cell_size));
            for (int v = 0; v < s.n_cameras && !keep; ++v) {
                const ss_pool_camera& c = s.cameras[v];
                double pc[3];
                cam_point(c, ctr, pc);
                const double x = pc[0], y = pc[1], z = pc[2], mg = s.margin;
                if (da(z, mg) < c.near_plane || ds(z, mg) > c.far_plane) continue;
                if (dm(ds(dm(z, c.tx), x), c.nx) < -mg || dm(da(dm(z, c.tx), x), c.nx) < -mg) continue;
                if (dm(ds(dm(z, c.ty), y), c.ny) < -mg || dm(da(dm(z, c.ty), y), c.ny) < -mg) continue;
                if (c.depth) {  // _center_depth_pass (expansion.py:95-107)
                    if (c.near_plane <= z && z <= c.far_plane) {
                        const double u = da(dd(dm(c.fx, x), z), c.cx), w = da(dd(dm(c.fy, y), z), c.cy);
                        const double fu = floor(u), fw = floor(w);
                        if (fu >= 0 && fu < c.width && fw >= 0 && fw < c.height) {
                            const double dz = c.depth[(int64_t)fw * c.width + (int64_t)fu];
                            if (!(z <= da(dz, mg))) continue;  // in the frustum and occluded
                        }
                    }
                }
                keep = true;
            }
        }
        flag[i] = keep;
    }
}

__global__ void k_scatter_rows(const uint8_t* __restrict__ flag, const uint64_t* __restrict__ pos, int64_t n,
                               const int64_t* __restrict__ row_ids, int64_t* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (flag[i]) out[pos[i]] = row_ids ? row_ids[i] : i;
}

// ---------------------------------------------------------------- gather
template <typename T>
__global__ void k_gather_col(const T* __restrict__ src, T* __restrict__ dst, const int64_t* __restrict__ map,
                             int64_t n_out, int width, const T* __restrict__ fill, int64_t fill_rows) {
    const int64_t total = n_out * width;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / width;
        const int k = (int)(e - i * width);
        const int64_t r = map[i];
        dst[e] = r >= 0 ? src[r * width + k] : fill[(-1 - r) % (fill_rows > 0 ? fill_rows : 1) * width + k];
    }
}

// ---------------------------------------------------------------- grid
__global__ void k_cells(const float* __restrict__ means, int64_t n, ss_grid_spec g, int64_t* __restrict__ cells,
                        unsigned long long* __restrict__ mm) {
    SS_PDL_WAIT();
    // per-axis min / max of the order-preserving offsets: thread -> warp -> one atomic per block and value
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t c[3];
        cell_of(means + 3 * i, g.origin, g.cell_size, c);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            cells[3 * i + k] = c[k];
            const unsigned long long o = (unsigned long long)(c[k] + (1ll << 62));
            lo[k] = o < lo[k] ? o : lo[k];
            hi[k] = o > hi[k] ? o : hi[k];
        }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo[k], off);
            const unsigned long long b = __shfl_xor_sync(0xffffffffu, hi[k], off);
            lo[k] = a < lo[k] ? a : lo[k];
            hi[k] = b > hi[k] ? b : hi[k];
        }
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if (lo[k] != ~0ull) atomicMin(&mm[k], lo[k]);
            if (hi[k]) atomicMax(&mm[3 + k], hi[k]);
        }
}

__global__ void k_cell_keys(const int64_t* __restrict__ cells, int64_t n, const unsigned long long* __restrict__ mm,
                            uint32_t* __restrict__ key, uint32_t* __restrict__ val) {
    const unsigned long long sy = mm[4] - mm[1] + 1, sz = mm[5] - mm[2] + 1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long x = (unsigned long long)(cells[3 * i] + (1ll << 62)) - mm[0];
        const unsigned long long y = (unsigned long long)(cells[3 * i + 1] + (1ll << 62)) - mm[1];
        const unsigned long long z = (unsigned long long)(cells[3 * i + 2] + (1ll << 62)) - mm[2];
        key[i] = (uint32_t)((x * sy + y) * sz + z);
        val[i] = (uint32_t)i;
    }
}

// group heads of the cell-sorted rows: head flag, and per group its first row
__global__ void k_group_heads(const uint32_t* __restrict__ key, const uint32_t* __restrict__ rows, int64_t n,
                              uint8_t* __restrict__ head) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        head[i] = i == 0 || key[i] != key[i - 1];
}

__global__ void k_group_info(const uint8_t* __restrict__ head, const uint64_t* __restrict__ gid, int64_t n,
                             const uint32_t* __restrict__ rows, uint32_t* __restrict__ gstart,
                             uint32_t* __restrict__ gfirst_row, uint32_t* __restrict__ gidx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (head[i]) {
            gstart[gid[i]] = (uint32_t)i;
            gfirst_row[gid[i]] = rows[i];  // stable sort: the group's smallest row
            gidx[gid[i]] = (uint32_t)gid[i];
        }
}

// cells in dict order: position p holds group gorder[p]
__global__ void k_group_len(const uint32_t* __restrict__ gstart, int64_t groups, int64_t n,
                            const uint32_t* __restrict__ gorder, uint32_t* __restrict__ len_ordered,
                            uint32_t* __restrict__ rank) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < groups; p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t g = gorder[p];
        const uint32_t end = g + 1 < groups ? gstart[g + 1] : (uint32_t)n;
        len_ordered[p] = end - gstart[g];
        rank[g] = (uint32_t)p;
    }
}

__global__ void k_grid_out(const uint8_t* __restrict__ head, const uint64_t* __restrict__ gid,
                           const uint32_t* __restrict__ gstart,
                           const uint32_t* __restrict__ rank, const uint64_t* __restrict__ out_off,
                           const uint32_t* __restrict__ rows, const int64_t* __restrict__ cells, int64_t n,
                           int64_t* __restrict__ cell_rows, int64_t* __restrict__ cell_keys,
                           int64_t* __restrict__ cell_lens, const uint32_t* __restrict__ len_ordered) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t g = gid[i] + head[i] - 1;
        const uint32_t p = rank[g];
        cell_rows[out_off[p] + (i - gstart[g])] = rows[i];
        if ((uint32_t)i == gstart[g]) {
#pragma unroll
            for (int k = 0; k < 3; ++k) cell_keys[3 * (int64_t)p + k] = cells[3 * (int64_t)rows[i] + k];
            cell_lens[p] = len_ordered[p];
        }
    }
}

// ---------------------------------------------------------------- zigzag varints
__global__ void k_zz_len(const int64_t* __restrict__ perm, int64_t n, uint8_t* __restrict__ len, uint64_t* __restrict__ zz) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t off = perm[i] - i;
        const uint64_t z = ((uint64_t)off << 1) ^ (uint64_t)(off >> 63);  // packets.py:155-156
        zz[i] = z;
        int l = 1;
        for (uint64_t v = z; v >= 0x80; v >>= 7) ++l;
        len[i] = (uint8_t)l;
    }
}

__global__ void k_zz_write(const uint64_t* __restrict__ zz, const uint64_t* __restrict__ pos, int64_t n,
                           uint8_t* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t v = zz[i];
        uint8_t* p = out + pos[i];
        while (v >= 0x80) {
            *p++ = (uint8_t)(v & 0x7F) | 0x80;
            v >>= 7;
        }
        *p = (uint8_t)v;
    }
}

}  // namespace

extern "C" {

int ss_select_rows(ss_ctx* ctx, const ss_select* s, int64_t* out, int64_t* count_out) {
    if (!ctx || !s || !out || !count_out) return SS_ERR_INVALID;
    if (s->kind < SS_SELECT_FREEZE || s->kind > SS_SELECT_PRECULL) return ss_fail(ctx, SS_ERR_INVALID, "bad select kind");
    SS_TRY(ss_scratch_reset(ctx));
    *count_out = 0;
    if (s->n <= 0) return SS_OK;
    cudaStream_t st = ctx->stream;
    uint8_t* flag = SS_SCRATCH(ctx, uint8_t, s->n);
    uint64_t* pos = SS_SCRATCH(ctx, uint64_t, s->n);
    uint64_t* tot = SS_SCRATCH(ctx, uint64_t, 1);
    if (!flag || !pos || !tot) return SS_ERR_CUDA;
    ss_select s2 = *s;
    if (s->kind == SS_SELECT_PRECULL) {  // camera array to device
        ss_pool_camera* cams = SS_SCRATCH(ctx, ss_pool_camera, s->n_cameras > 0 ? s->n_cameras : 1);
        if (!cams) return SS_ERR_CUDA;
        SS_CUDA(ctx, cudaMemcpyAsync(cams, s->cameras, sizeof(ss_pool_camera) * s->n_cameras, cudaMemcpyHostToDevice, st));
        s2.cameras = cams;
    }
    k_select_flags<<<grid_for(ctx, s->n), 256, 0, st>>>(s2, flag);
    SS_CHECK_LAUNCH(ctx);
    SS_TRY(ss_scan_u8_to_u64(ctx, flag, pos, s->n, tot));
    k_scatter_rows<<<grid_for(ctx, s->n), 256, 0, st>>>(flag, pos, s->n, s->row_ids, out);
    SS_CHECK_LAUNCH(ctx);
    uint64_t c = 0;
    SS_TRY(ss_read_u64(ctx, tot, &c));  // synchronises (the caller needs the count)
    *count_out = (int64_t)c;
    return SS_OK;
}

int ss_gather_rows(ss_ctx* ctx, const ss_model* src, ss_model* dst, const int64_t* map, int64_t n_out,
                   const ss_model* fill) {
    if (!ctx || !src || !dst || (n_out > 0 && !map)) return SS_ERR_INVALID;
    if (src->sh_degree != dst->sh_degree) return ss_fail(ctx, SS_ERR_INVALID, "sh_degree mismatch");
    if (n_out == 0) return SS_OK;
    cudaStream_t s = ctx->stream;
    const int B = (src->sh_degree + 1) * (src->sh_degree + 1);
    const int64_t fr = fill ? fill->count : 0;
    const int g = grid_for(ctx, n_out * 3 * B);
    k_gather_col<float><<<g, 256, 0, s>>>(src->means, dst->means, map, n_out, 3, fill ? fill->means : nullptr, fr);
    k_gather_col<float><<<g, 256, 0, s>>>(src->log_scales, dst->log_scales, map, n_out, 3, fill ? fill->log_scales : nullptr, fr);
    k_gather_col<float><<<g, 256, 0, s>>>(src->quaternions, dst->quaternions, map, n_out, 4, fill ? fill->quaternions : nullptr, fr);
    k_gather_col<float><<<g, 256, 0, s>>>(src->logit_opacities, dst->logit_opacities, map, n_out, 1,
                                          fill ? fill->logit_opacities : nullptr, fr);
    k_gather_col<float><<<g, 256, 0, s>>>(src->sh_coeffs, dst->sh_coeffs, map, n_out, 3 * B, fill ? fill->sh_coeffs : nullptr, fr);
    k_gather_col<float><<<g, 256, 0, s>>>(src->light_visibility, dst->light_visibility, map, n_out, 1,
                                          fill ? fill->light_visibility : nullptr, fr);
    k_gather_col<int32_t><<<g, 256, 0, s>>>(src->object_ids, dst->object_ids, map, n_out, 1, fill ? fill->object_ids : nullptr, fr);
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}

int ss_grid_rebuild(ss_ctx* ctx, const float* means, int64_t n, const ss_grid_spec* g, int64_t* cells,
                    int64_t* cell_keys, int64_t* cell_lens, int64_t* cell_rows, int64_t* n_cells) {
    if (!ctx || !g || !n_cells || (n > 0 && (!means || !cells || !cell_keys || !cell_lens || !cell_rows)))
        return SS_ERR_INVALID;
    if (!(g->cell_size > 0)) return ss_fail(ctx, SS_ERR_INVALID, "cell_size must be positive");
    SS_TRY(ss_scratch_reset(ctx));
    *n_cells = 0;
    if (n == 0) return SS_OK;
    if (n > 0xfffffffell) return ss_fail(ctx, SS_ERR_CAPACITY, "grid rebuild limited to 2^32 rows");
    cudaStream_t s = ctx->stream;
    unsigned long long* mm = SS_SCRATCH(ctx, unsigned long long, 6);
    uint32_t* key = SS_SCRATCH(ctx, uint32_t, n);
    uint32_t* val = SS_SCRATCH(ctx, uint32_t, n);
    uint32_t* k2 = SS_SCRATCH(ctx, uint32_t, n);
    uint32_t* v2 = SS_SCRATCH(ctx, uint32_t, n);
    uint8_t* head = SS_SCRATCH(ctx, uint8_t, n);
    uint64_t* gid = SS_SCRATCH(ctx, uint64_t, n);
    uint64_t* tot = SS_SCRATCH(ctx, uint64_t, 1);
    if (!mm || !key || !val || !k2 || !v2 || !head || !gid || !tot) return SS_ERR_CUDA;
    unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0, 0, 0};
    SS_CUDA(ctx, cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, s));
    k_cells<<<grid_for(ctx, n), 256, 0, s>>>(means, n, *g, cells, mm);
    SS_CHECK_LAUNCH(ctx);
    unsigned long long hm[6];
    SS_CUDA(ctx, cudaMemcpyAsync(hm, mm, sizeof(hm), cudaMemcpyDeviceToHost, s));
    SS_CUDA(ctx, ss_stream_sync(ctx));
    const double span = (double)(hm[3] - hm[0] + 1) * (double)(hm[4] - hm[1] + 1) * (double)(hm[5] - hm[2] + 1);
    if (span > 4294967295.0) return ss_fail(ctx, SS_ERR_CAPACITY, "grid spans more than 2^32 cells");
    int bits = 1;
    while (bits < 32 && (double)(1ull << bits) < span) ++bits;
    k_cell_keys<<<grid_for(ctx, n), 256, 0, s>>>(cells, n, mm, key, val);
    SS_CHECK_LAUNCH(ctx);
    SS_TRY(ss_radix_sort_u32(ctx, key, val, k2, v2, n, bits));  // stable: rows ascending within a cell
    k_group_heads<<<grid_for(ctx, n), 256, 0, s>>>(key, val, n, head);
    SS_CHECK_LAUNCH(ctx);
    SS_TRY(ss_scan_u8_to_u64(ctx, head, gid, n, tot));
    uint64_t G = 0;
    SS_TRY(ss_read_u64(ctx, tot, &G));
    // gid is the exclusive scan of the head flags: element i belongs to group gid[i] + head[i] - 1
    uint32_t* gstart = SS_SCRATCH(ctx, uint32_t, G);
    uint32_t* gfirst = SS_SCRATCH(ctx, uint32_t, G);
    uint32_t* gidx = SS_SCRATCH(ctx, uint32_t, G);
    uint32_t* gf2 = SS_SCRATCH(ctx, uint32_t, G);
    uint32_t* gi2 = SS_SCRATCH(ctx, uint32_t, G);
    uint32_t* lens = SS_SCRATCH(ctx, uint32_t, G);
    uint32_t* rank = SS_SCRATCH(ctx, uint32_t, G);
    uint64_t* off = SS_SCRATCH(ctx, uint64_t, G);
    if (!gstart || !gfirst || !gidx || !gf2 || !gi2 || !lens || !rank || !off) return SS_ERR_CUDA;
    k_group_info<<<grid_for(ctx, n), 256, 0, s>>>(head, gid, n, val, gstart, gfirst, gidx);
    SS_CHECK_LAUNCH(ctx);
    // dict order: groups by their first row (first appearance in row order)
    int rbits = 1;
    while (rbits < 32 && (1ull << rbits) < (unsigned long long)n) ++rbits;
    SS_TRY(ss_radix_sort_u32(ctx, gfirst, gidx, gf2, gi2, (int64_t)G, rbits));
    k_group_len<<<grid_for(ctx, G), 256, 0, s>>>(gstart, (int64_t)G, n, gidx, lens, rank);
    SS_CHECK_LAUNCH(ctx);
    SS_TRY(ss_scan_u32_to_u64(ctx, lens, off, (int64_t)G, tot));
    k_grid_out<<<grid_for(ctx, n), 256, 0, s>>>(head, gid, gstart, rank, off, val, cells, n, cell_rows, cell_keys,
                                                cell_lens, lens);
    SS_CHECK_LAUNCH(ctx);
    *n_cells = (int64_t)G;
    return SS_OK;
}

int ss_zigzag_varints(ss_ctx* ctx, const int64_t* perm, int64_t n, uint8_t* out, uint64_t out_cap, uint64_t* len_out) {
    if (!ctx || !len_out || (n > 0 && (!perm || !out))) return SS_ERR_INVALID;
    SS_TRY(ss_scratch_reset(ctx));
    *len_out = 0;
    if (n == 0) return SS_OK;
    cudaStream_t s = ctx->stream;
    uint8_t* len = SS_SCRATCH(ctx, uint8_t, n);
    uint64_t* zz = SS_SCRATCH(ctx, uint64_t, n);
    uint64_t* pos = SS_SCRATCH(ctx, uint64_t, n);
    uint64_t* tot = SS_SCRATCH(ctx, uint64_t, 1);
    if (!len || !zz || !pos || !tot) return SS_ERR_CUDA;
    k_zz_len<<<grid_for(ctx, n), 256, 0, s>>>(perm, n, len, zz);
    SS_CHECK_LAUNCH(ctx);
    SS_TRY(ss_scan_u8_to_u64(ctx, len, pos, n, tot));
    uint64_t total = 0;
    SS_TRY(ss_read_u64(ctx, tot, &total));
    if (total > out_cap) return ss_fail(ctx, SS_ERR_CAPACITY, "varint output too small");
    k_zz_write<<<grid_for(ctx, n), 256, 0, s>>>(zz, pos, n, out);
    SS_CHECK_LAUNCH(ctx);
    *len_out = total;
    return SS_OK;
}

}  // extern "C"
