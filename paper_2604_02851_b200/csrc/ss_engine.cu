// Ray-cast scene engine (the game-engine stand-in that
// produces the ground truth and the expansion inputs), one thread per pixel:
//
//   ref engine.py:88-127  trace            nearest hit over every object
//   ref engine.py:130-137 light_occluded   any-hit shadow ray from p + 1e-5 n
//   ref engine.py:140-148 shade            albedo (ambient + I max(0, n.-l) lit)
//   ref engine.py:151-158 render_ground_truth
//   ref engine.py:161-189 capture_input_buffers
//   ref engine.py:192-205 render_depth / render_ortho_depth
//   ref scene.py:28-137   Plane / Sphere / Box intersect, scene.py:140-161 Albedo
//
// Arithmetic is float64 and mirrors the reference op for op: elementwise
// steps use explicit round-to-nearest intrinsics (no contraction), 3-term
// sums are ((a + b) + c) as numpy's reductions, and every `@` follows the
// FMA pattern numpy's matmul produced for that operand layout (measured
// against numpy in tests/golden/make_golden.py::engine_cases):
//   (N,3) @ (3,3)            fma(x2,y2, fma(x1,y1, x0 y0))       "D"
//   (N,3) @ (3,), N >= 2      fma(x2,y2, fma(x0,y0, x1 y1))       "C"
//   broadcast rows @ (3,)     ((x0 y0 + x1 y1) + x2 y2)            "S"
// (broadcast rows: the shadow rays' and the ortho rays' shared direction).
#include <math.h>

#include "ss_internal.cuh"

namespace {

constexpr int EN_THREADS = 128;

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ double dotD(const double* x, double y0, double y1, double y2) {
    return __fma_rn(x[2], y2, __fma_rn(x[1], y1, mul(x[0], y0)));
}
__device__ __forceinline__ double dotC(const double* x, const double* y) {
    return __fma_rn(x[2], y[2], __fma_rn(x[0], y[0], mul(x[1], y[1])));
}
__device__ __forceinline__ double dotS(const double* x, const double* y) {
    return add(add(mul(x[0], y[0]), mul(x[1], y[1])), mul(x[2], y[2]));
}
// numpy.minimum / maximum (NaN propagates)
__device__ __forceinline__ double np_min(double a, double b) { return isnan(a) || isnan(b) ? NAN : (a <= b ? a : b); }
__device__ __forceinline__ double np_max(double a, double b) { return isnan(a) || isnan(b) ? NAN : (a >= b ? a : b); }

// x @ R (row vector times matrix, (N,3)@(3,3))
__device__ __forceinline__ void vec_mat(const double* x, const double* R, double* out) {
#pragma unroll
    for (int j = 0; j < 3; ++j) out[j] = dotD(x, R[j], R[3 + j], R[6 + j]);
}
// x @ R.T
__device__ __forceinline__ void vec_matT(const double* x, const double* R, double* out) {
#pragma unroll
    for (int j = 0; j < 3; ++j) out[j] = dotD(x, R[3 * j], R[3 * j + 1], R[3 * j + 2]);
}

struct Isect {
    double t;         // inf: miss
    double n0, n1, n2;  // local normal
};

// one object's hit distance and local normal; ref scene.py
__device__ __forceinline__ Isect intersect(const ss_scene_object& ob, const double* o, const double* d, bool d_bcast) {
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    Isect r;
    if (ob.shape == SS_SHAPE_PLANE) {  // scene.py:48-68
        const double* nn = ob.b;
        const double denom = d_bcast ? dotS(d, nn) : dotC(d, nn);
        double pm[3] = {sub(ob.a[0], o[0]), sub(ob.a[1], o[1]), sub(ob.a[2], o[2])};
        double t = dvd(dotC(pm, nn), denom);
        if (!(fabs(denom) > 1e-12)) t = INF;
        if (!(t > 1e-9)) t = INF;
        if (ob.has_extent) {
            const double tt = isfinite(t) ? t : 0.0;
            const double rel[3] = {sub(add(o[0], mul(tt, d[0])), ob.a[0]), sub(add(o[1], mul(tt, d[1])), ob.a[1]),
                                   sub(add(o[2], mul(tt, d[2])), ob.a[2])};
            const bool inside = fabs(dotC(rel, ob.u)) <= ob.extent[0] && fabs(dotC(rel, ob.v)) <= ob.extent[1];
            if (!inside) t = INF;
        }
        const bool flip = denom > 0.0;
        r.t = t;
        r.n0 = flip ? -nn[0] : nn[0];
        r.n1 = flip ? -nn[1] : nn[1];
        r.n2 = flip ? -nn[2] : nn[2];
        return r;
    }
    if (ob.shape == SS_SHAPE_SPHERE) {  // scene.py:80-95
        const double oc[3] = {sub(o[0], ob.a[0]), sub(o[1], ob.a[1]), sub(o[2], ob.a[2])};
        const double b = add(add(mul(oc[0], d[0]), mul(oc[1], d[1])), mul(oc[2], d[2]));
        const double c = sub(add(add(mul(oc[0], oc[0]), mul(oc[1], oc[1])), mul(oc[2], oc[2])), mul(ob.radius, ob.radius));
        const double disc = sub(mul(b, b), c);
        const double sq = __dsqrt_rn(np_max(disc, 0.0));
        const double t0 = sub(-b, sq), t1 = add(-b, sq);
        double t = t0 > 1e-9 ? t0 : (t1 > 1e-9 ? t1 : INF);
        if (!(disc >= 0.0)) t = INF;
        const bool hit = isfinite(t);
        r.t = t;
        r.n0 = hit ? dvd(sub(add(o[0], mul(t, d[0])), ob.a[0]), ob.radius) : 0.0;
        r.n1 = hit ? dvd(sub(add(o[1], mul(t, d[1])), ob.a[1]), ob.radius) : 0.0;
        r.n2 = hit ? dvd(sub(add(o[2], mul(t, d[2])), ob.a[2]), ob.radius) : 0.0;
        return r;
    }
    // box, scene.py:110-130
    double tn = 0.0, tf = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double inv = dvd(1.0, d[k]);
        const double lo = sub(ob.a[k], ob.b[k]), hi = add(ob.a[k], ob.b[k]);
        const double tl = mul(sub(lo, o[k]), inv), th = mul(sub(hi, o[k]), inv);
        const double a1 = np_min(tl, th), a2 = np_max(tl, th);
        tn = k ? np_max(tn, a1) : a1;
        tf = k ? np_min(tf, a2) : a2;
    }
    const double t = (tn <= tf && tf > 1e-9) ? (tn > 1e-9 ? tn : tf) : INF;
    r.t = t;
    r.n0 = r.n1 = r.n2 = 0.0;
    if (isfinite(t)) {
        const double x = dvd(sub(add(o[0], mul(t, d[0])), ob.a[0]), ob.b[0]);
        const double y = dvd(sub(add(o[1], mul(t, d[1])), ob.a[1]), ob.b[1]);
        const double z = dvd(sub(add(o[2], mul(t, d[2])), ob.a[2]), ob.b[2]);
        // argmax |rel| (first on ties), then its sign
        const bool ay = fabs(y) > fabs(x);
        const double m = ay ? y : x;
        const bool az = fabs(z) > fabs(m);
        const double v = az ? z : m;
        const double sg = v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0);
        r.n0 = (!ay && !az) ? sg : 0.0;
        r.n1 = (ay && !az) ? sg : 0.0;
        r.n2 = az ? sg : 0.0;
    }
    return r;
}

// ray in an object's local frame (trace: engine.py:99-108)
__device__ __forceinline__ void to_local(const ss_scene_object& ob, const double* o, const double* d, double* ol, double* dl) {
    const double om[3] = {sub(o[0], ob.t[0]), sub(o[1], ob.t[1]), sub(o[2], ob.t[2])};
    vec_mat(om, ob.R, ol);
    vec_mat(d, ob.R, dl);
}

struct Hit {
    double t;
    int k;
    double nl[3], pl[3];  // local normal and point of the nearest hit
};

__device__ Hit trace_nearest(const ss_scene_object* objs, int n_obj, const double* o, const double* d, bool d_bcast) {
    Hit h;
    h.t = __longlong_as_double(0x7ff0000000000000ll);
    h.k = -1;
#pragma unroll 1
    for (int k = 0; k < n_obj; ++k) {
        const ss_scene_object& ob = objs[k];
        double ol[3], dl[3];
        const double* oo = o;
        const double* dd = d;
        bool bc = d_bcast;
        if (ob.has_transform) {
            to_local(ob, o, d, ol, dl);
            oo = ol, dd = dl, bc = false;  // d @ R is a fresh contiguous array
        }
        const Isect r = intersect(ob, oo, dd, bc);
        if (r.t < h.t) {
            h.t = r.t;
            h.k = k;
            h.nl[0] = r.n0, h.nl[1] = r.n1, h.nl[2] = r.n2;
#pragma unroll
            for (int j = 0; j < 3; ++j) h.pl[j] = add(oo[j], mul(r.t, dd[j]));
        }
    }
    return h;
}

__device__ bool trace_any(const ss_scene_object* objs, int n_obj, const double* o, const double* d) {
#pragma unroll 1
    for (int k = 0; k < n_obj; ++k) {
        const ss_scene_object& ob = objs[k];
        double ol[3], dl[3];
        double tk;
        if (ob.has_transform) {
            to_local(ob, o, d, ol, dl);
            tk = intersect(ob, ol, dl, false).t;
        } else {
            tk = intersect(ob, o, d, true).t;
        }
        if (tk < __longlong_as_double(0x7ff0000000000000ll)) return true;
    }
    return false;
}

// Albedo.eval (scene.py:152-158)
__device__ __forceinline__ void albedo_eval(const ss_scene_object& ob, const double* pl, const double* nl, double* c) {
    if (ob.albedo_kind == 0) {
#pragma unroll
        for (int j = 0; j < 3; ++j) c[j] = ob.color[j];
        return;
    }
    double f[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) f[j] = floor(dvd(add(pl[j], mul(1e-6, nl[j])), ob.scale));
    const long long s = (long long)add(add(f[0], f[1]), f[2]);
    const double* src = (s & 1) == 0 ? ob.color : ob.color2;
#pragma unroll
    for (int j = 0; j < 3; ++j) c[j] = src[j];
}

__device__ __forceinline__ double clip01(double x) { return np_min(np_max(x, 0.0), 1.0); }

struct SceneArgs {
    const ss_scene_object* objs;
    int n_obj;
    double neg_l[3];  // -light.direction
    double intensity[3], ambient[3], background[3];
};

__global__ void __launch_bounds__(EN_THREADS) k_engine(SceneArgs S, ss_engine_camera cam, ss_engine_out out) {
    SS_PDL_WAIT();
    extern __shared__ ss_scene_object s_obj[];
    for (int k = threadIdx.x; k < S.n_obj; k += blockDim.x) s_obj[k] = S.objs[k];
    __syncthreads();
    const int64_t npx = (int64_t)cam.width * cam.height;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npx) return;
    const int i = (int)(p % cam.width), jrow = (int)(p / cam.width);
    double o[3], d[3];
    const double* R = cam.R;
    bool d_bcast;
    if (cam.kind == 0) {  // camera_rays (geometry.py:238-249)
        const double x = dvd(sub(add((double)i, 0.5), cam.cx), cam.fx);
        const double y = dvd(sub(add((double)jrow, 0.5), cam.cy), cam.fy);
        const double dc[3] = {x, y, 1.0};
        vec_matT(dc, R, d);
        const double nrm = __dsqrt_rn(add(add(mul(d[0], d[0]), mul(d[1], d[1])), mul(d[2], d[2])));
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            d[k] = dvd(d[k], nrm);
            o[k] = cam.position[k];
        }
        d_bcast = false;
    } else if (cam.kind == 2) {  // explicit rays (trace, engine.py:88): origins broadcast against dirs
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            o[k] = cam.ray_origins[(int64_t)cam.origin_stride * p + k];
            d[k] = cam.ray_dirs[(int64_t)cam.dir_stride * p + k];
        }
        d_bcast = cam.dir_stride == 0;
    } else {  // OrthoCamera.pixel_origins (geometry.py:273-281), rays along +Z
        const double u = dvd(add((double)i, 0.5), (double)cam.width);
        const double v = dvd(add((double)jrow, 0.5), (double)cam.height);
        const double pc[3] = {mul(sub(mul(u, 2.0), 1.0), cam.half_width), mul(sub(mul(v, 2.0), 1.0), cam.half_height), 0.0};
        vec_matT(pc, R, o);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            o[k] = add(o[k], cam.position[k]);
            d[k] = R[3 * k + 2];  // pose.forward() = R[:, 2]
        }
        d_bcast = true;
    }
    const Hit h = trace_nearest(s_obj, S.n_obj, o, d, d_bcast);
    const bool valid = isfinite(h.t);
    const double tt = valid ? h.t : 0.0;
    double wp[3], nw[3] = {0.0, 0.0, 0.0}, alb[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < 3; ++k) wp[k] = add(o[k], mul(tt, d[k]));
    if (valid) {
        const ss_scene_object& ob = s_obj[h.k];
        albedo_eval(ob, h.pl, h.nl, alb);
        if (ob.has_transform) vec_matT(h.nl, ob.R, nw);
        else nw[0] = h.nl[0], nw[1] = h.nl[1], nw[2] = h.nl[2];
    }
    if (out.depth_or_far) {
        double z;
        if (cam.kind == 0) {  // render_depth: (wp - pos) @ forward
            const double rel[3] = {sub(wp[0], cam.position[0]), sub(wp[1], cam.position[1]), sub(wp[2], cam.position[2])};
            const double fw[3] = {R[2], R[5], R[8]};
            z = dotC(rel, fw);
        } else {
            z = h.t;  // render_ortho_depth: the ray parameter
        }
        out.depth_or_far[p] = valid ? z : cam.far;
    }
    const bool need_shade = out.gt_f32 || out.gt_f64 || out.shaded || out.lit;
    if (need_shade) {
        bool lit = false;
        if (valid) {  // light_occluded (engine.py:130-137)
            const double so[3] = {add(wp[0], mul(1e-5, nw[0])), add(wp[1], mul(1e-5, nw[1])), add(wp[2], mul(1e-5, nw[2]))};
            lit = !trace_any(s_obj, S.n_obj, so, S.neg_l);
        }
        const double cs = np_max(0.0, dotC(nw, S.neg_l));
        const double cl = mul(cs, lit ? 1.0 : 0.0);
        double col[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) col[k] = clip01(mul(alb[k], add(S.ambient[k], mul(S.intensity[k], cl))));
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double g = clip01(valid ? col[k] : S.background[k]);
            if (out.gt_f64) out.gt_f64[3 * p + k] = g;
            if (out.gt_f32) out.gt_f32[3 * p + k] = (float)g;
            if (out.shaded) out.shaded[3 * p + k] = g;
        }
        if (out.lit) out.lit[p] = valid && lit;
    }
    if (out.t) out.t[p] = h.t;
    if (out.object_index) out.object_index[p] = h.k;
    if (out.valid) out.valid[p] = valid;
    if (out.world_pos)
        for (int k = 0; k < 3; ++k) out.world_pos[3 * p + k] = valid ? wp[k] : 0.0;
    if (out.normal)
        for (int k = 0; k < 3; ++k) out.normal[3 * p + k] = valid ? nw[k] : 0.0;
    if (out.albedo)
        for (int k = 0; k < 3; ++k) out.albedo[3 * p + k] = valid ? alb[k] : 0.0;
    if (out.object_id) out.object_id[p] = valid ? s_obj[h.k].object_id : 0;
    if (out.depth || out.footprint) {  // capture_input_buffers (engine.py:166-168)
        const double rel[3] = {sub(wp[0], cam.position[0]), sub(wp[1], cam.position[1]), sub(wp[2], cam.position[2])};
        const double fw[3] = {R[2], R[5], R[8]};
        const double z = valid ? dotC(rel, fw) : 0.0;
        if (out.depth) out.depth[p] = z;
        if (out.footprint) out.footprint[p] = valid ? mul(z, cam.footprint_scale) : 0.0;
    }
}

}  // namespace

extern "C" int ss_engine_render(ss_ctx* ctx, const ss_scene* scene, const ss_engine_camera* cam, const ss_engine_out* out) {
    if (!ctx || !scene || !cam || !out) return SS_ERR_INVALID;
    if (cam->width < 1 || cam->height < 1 || cam->kind < 0 || cam->kind > 2) return ss_fail(ctx, SS_ERR_INVALID, "bad camera");
    if (cam->kind == 2 && (!cam->ray_origins || !cam->ray_dirs || cam->height != 1 ||
                           (cam->origin_stride != 0 && cam->origin_stride != 3) || (cam->dir_stride != 0 && cam->dir_stride != 3)))
        return ss_fail(ctx, SS_ERR_INVALID, "rays: device origins/dirs with stride 0 or 3, height 1");
    if (scene->n_objects < 0 || scene->n_objects > 256 || (scene->n_objects && !scene->objects))
        return ss_fail(ctx, SS_ERR_INVALID, "0..256 scene objects");
    for (int k = 0; k < scene->n_objects; ++k) {
        const ss_scene_object& ob = scene->objects[k];
        if (ob.shape < 0 || ob.shape > 2 || ob.albedo_kind < 0 || ob.albedo_kind > 1)
            return ss_fail(ctx, SS_ERR_INVALID, "object %d: unknown shape or albedo kind", k);
    }
    SS_TRY(ss_scratch_reset(ctx));
    SceneArgs S;
    S.n_obj = scene->n_objects;
    S.objs = nullptr;
    if (S.n_obj) {
        ss_scene_object* d = SS_SCRATCH(ctx, ss_scene_object, S.n_obj);
        if (!d) return SS_ERR_CUDA;
        SS_CUDA(ctx, cudaMemcpyAsync(d, scene->objects, sizeof(ss_scene_object) * S.n_obj, cudaMemcpyHostToDevice, ctx->stream));
        S.objs = d;
    }
    for (int k = 0; k < 3; ++k) {
        S.neg_l[k] = -scene->light_direction[k];
        S.intensity[k] = scene->light_intensity[k];
        S.ambient[k] = scene->ambient[k];
        S.background[k] = scene->background[k];
    }
    const int64_t npx = (int64_t)cam->width * cam->height;
    const size_t smem = sizeof(ss_scene_object) * (size_t)S.n_obj;
    if (smem > 48 * 1024)
        SS_CUDA(ctx, cudaFuncSetAttribute(k_engine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SS_CUDA(ctx, ss_launch((k_engine), dim3((unsigned)((npx + EN_THREADS - 1) / EN_THREADS)), dim3(EN_THREADS), smem, ctx->stream,
                           S, *cam, *out));
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}
