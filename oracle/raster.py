"""CPU restatement of the splatstream differentiable renderer (test infrastructure only).

Reference behaviour followed (file:line under /root/reference/pkg/src/splatstream):
  sh basis / gradient        render.py:63-136
  normal proxy (5e-3 margin) render.py:139-151
  shading core               render.py:175-197
  preprocess                 render.py:226-290  (prepare_splats)
  rectangular window         render.py:293-301  (splat_window)
  alpha / composite          render.py:304-336  (T-gate before the splat,
                                                 alpha cap 0.999, [0,1] colour clamp)
  backward                   optim.py:113-268   (front-to-back, S = C - prefix - contrib)

Two deliberate definitions, shared op-for-op with the CUDA preprocess kernel so
that depth keys, windows, tile lists and tile ranges are bit-identical between
this oracle and the GPU:
  * ``det_exp`` -- a deterministic exp built only from IEEE-exact operations
    (used for exp(2*log_scale)); numpy's and CUDA's libm exps differ by an ulp.
  * the summation order of every small matrix product is written out below.
Agreement of these windows/orders with the reference's own numpy/BLAS values
is measured by tests/test_oracle_golden.py (expected 100%).
All arithmetic is float64.
"""

from __future__ import annotations

import numpy as np

SH_C0 = 0.2820947918
SH_C1 = 0.4886025119
SH_C2 = (1.0925484306, -1.0925484306, 0.3153915653, -1.0925484306, 0.5462742153)
SH_C3 = (-0.5900435899, 2.8906114426, -0.4570457995, 0.3731763326,
         -0.4570457995, 1.4453057213, -0.5900435899)
T_CUTOFF = 1e-4
ALPHA_CAP = 0.999
BLUR = 0.3
AXIS_MARGIN = 5e-3
TILE = 16

# ---------------------------------------------------------------- det_exp
_LN2_HI = 6.93147180369123816490e-01  # fdlibm split: k*_LN2_HI exact for |k| < 2^11
_LN2_LO = 1.90821492927058770002e-10
_INV_LN2 = 1.44269504088896338700e+00
_EXP_TAYLOR = [1.0 / float(np.prod(np.arange(1, k + 1, dtype=np.float64))) for k in range(14)]


def det_exp(x):
    """exp(x) from IEEE-exact ops only: k = rint(x/ln2), r = x - k ln2 (two-part),
    degree-13 Taylor in Horner form, scale by 2^k.  Mirrored by ss_det_exp()
    in csrc/ss_math.cuh; ~1 ulp accurate on the range log-scales reach."""
    x = np.asarray(x, np.float64)
    k = np.rint(x * _INV_LN2)
    r = (x - k * _LN2_HI) - k * _LN2_LO
    p = np.full_like(r, _EXP_TAYLOR[13])
    for c in reversed(_EXP_TAYLOR[:13]):
        p = p * r + c
    return np.ldexp(p, k.astype(np.int64))


# ---------------------------------------------------------------- geometry
def quat_rotmat(q, norm_like_numpy=False):
    """(..., 4) wxyz -> (..., 3, 3), normalising first (ref geometry.py:53-60).
    Gaussians: explicit ((w^2+x^2)+y^2)+z^2 norm (mirrored by the kernel);
    cameras (norm_like_numpy): np.linalg.norm as the host code computes it."""
    q = np.asarray(q, np.float64)
    if norm_like_numpy:
        q = q / np.linalg.norm(q, axis=-1, keepdims=True)
        w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    else:
        w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
        n = np.sqrt(((w * w + x * x) + y * y) + z * z)
        w, x, y, z = w / n, x / n, y / n, z / n
    R = np.empty(q.shape[:-1] + (3, 3))
    R[..., 0, 0] = 1.0 - 2.0 * (y * y + z * z)
    R[..., 0, 1] = 2.0 * (x * y - w * z)
    R[..., 0, 2] = 2.0 * (x * z + w * y)
    R[..., 1, 0] = 2.0 * (x * y + w * z)
    R[..., 1, 1] = 1.0 - 2.0 * (x * x + z * z)
    R[..., 1, 2] = 2.0 * (y * z - w * x)
    R[..., 2, 0] = 2.0 * (x * z - w * y)
    R[..., 2, 1] = 2.0 * (y * z + w * x)
    R[..., 2, 2] = 1.0 - 2.0 * (x * x + y * y)
    return R


def drot_dquat(q):
    """dR/dq (M,4,3,3) for raw quaternions incl. normalisation (ref optim.py:87-110)."""
    q = np.asarray(q, np.float64)
    n = np.sqrt(((q[:, 0] ** 2 + q[:, 1] ** 2) + q[:, 2] ** 2) + q[:, 3] ** 2)
    u = q / n[:, None]
    w, x, y, z = u.T
    zero = np.zeros_like(w)
    dunit = np.empty((q.shape[0], 4, 3, 3))
    rows = {
        0: [[zero, -z, y], [z, zero, -x], [-y, x, zero]],
        1: [[zero, y, z], [y, -2 * x, -w], [z, w, -2 * x]],
        2: [[-2 * y, x, w], [x, zero, z], [-w, z, -2 * y]],
        3: [[-2 * z, -w, x], [w, -2 * z, y], [x, y, zero]],
    }
    for c, mat in rows.items():
        for i in range(3):
            for j in range(3):
                dunit[:, c, i, j] = 2.0 * mat[i][j]
    P = (np.eye(4)[None] - u[:, :, None] * u[:, None, :]) / n[:, None, None]  # dU_a/dq_k = P[k,a]
    return np.einsum("mka,maij->mkij", P, dunit)


def camera(pose, intr):
    """Flatten a pose/intrinsics pair into the numbers the kernels use."""
    R = quat_rotmat(np.asarray(pose.quaternion, np.float64), norm_like_numpy=True)
    fy = (intr.height / 2.0) / np.tan(intr.fov_y / 2.0)
    return dict(pos=np.asarray(pose.position, np.float64), R=R, W=intr.width, H=intr.height,
                fx=fy, fy=fy, cx=intr.width / 2.0, cy=intr.height / 2.0, near=intr.near)


# ---------------------------------------------------------------- SH
def sh_basis(d, degree):
    d = np.asarray(d, np.float64)
    B = (degree + 1) ** 2
    Y = np.empty(d.shape[:-1] + (B,))
    Y[..., 0] = SH_C0
    if degree < 1:
        return Y
    x, y, z = d[..., 0], d[..., 1], d[..., 2]
    Y[..., 1], Y[..., 2], Y[..., 3] = -SH_C1 * y, SH_C1 * z, -SH_C1 * x
    if degree < 2:
        return Y
    xx, yy, zz = x * x, y * y, z * z
    Y[..., 4] = SH_C2[0] * (x * y)
    Y[..., 5] = SH_C2[1] * (y * z)
    Y[..., 6] = SH_C2[2] * (2 * zz - xx - yy)
    Y[..., 7] = SH_C2[3] * (x * z)
    Y[..., 8] = SH_C2[4] * (xx - yy)
    if degree < 3:
        return Y
    Y[..., 9] = SH_C3[0] * y * (3 * xx - yy)
    Y[..., 10] = SH_C3[1] * (x * y) * z
    Y[..., 11] = SH_C3[2] * y * (4 * zz - xx - yy)
    Y[..., 12] = SH_C3[3] * z * (2 * zz - 3 * xx - 3 * yy)
    Y[..., 13] = SH_C3[4] * x * (4 * zz - xx - yy)
    Y[..., 14] = SH_C3[5] * z * (xx - yy)
    Y[..., 15] = SH_C3[6] * x * (xx - yy - 3 * zz)
    return Y


def sh_basis_jac(d, degree):
    """dY_b/dd_k, shape (..., B, 3)."""
    d = np.asarray(d, np.float64)
    B = (degree + 1) ** 2
    g = np.zeros(d.shape[:-1] + (B, 3))
    if degree < 1:
        return g
    x, y, z = d[..., 0], d[..., 1], d[..., 2]
    g[..., 1, 1], g[..., 2, 2], g[..., 3, 0] = -SH_C1, SH_C1, -SH_C1
    if degree >= 2:
        a, b, c, e, f = SH_C2
        g[..., 4, 0], g[..., 4, 1] = a * y, a * x
        g[..., 5, 1], g[..., 5, 2] = b * z, b * y
        g[..., 6, 0], g[..., 6, 1], g[..., 6, 2] = -2 * c * x, -2 * c * y, 4 * c * z
        g[..., 7, 0], g[..., 7, 2] = e * z, e * x
        g[..., 8, 0], g[..., 8, 1] = 2 * f * x, -2 * f * y
    if degree >= 3:
        c0, c1, c2, c3, c4, c5, c6 = SH_C3
        g[..., 9, 0], g[..., 9, 1] = c0 * 6 * x * y, c0 * (3 * x * x - 3 * y * y)
        g[..., 10, 0], g[..., 10, 1], g[..., 10, 2] = c1 * y * z, c1 * x * z, c1 * x * y
        g[..., 11, 0] = c2 * (-2 * x * y)
        g[..., 11, 1] = c2 * (4 * z * z - x * x - 3 * y * y)
        g[..., 11, 2] = c2 * (8 * y * z)
        g[..., 12, 0], g[..., 12, 1] = c3 * (-6 * x * z), c3 * (-6 * y * z)
        g[..., 12, 2] = c3 * (6 * z * z - 3 * x * x - 3 * y * y)
        g[..., 13, 0] = c4 * (4 * z * z - 3 * x * x - y * y)
        g[..., 13, 1], g[..., 13, 2] = c4 * (-2 * x * y), c4 * (8 * x * z)
        g[..., 14, 0], g[..., 14, 1] = c5 * (2 * x * z), c5 * (-2 * y * z)
        g[..., 14, 2] = c5 * (x * x - y * y)
        g[..., 15, 0] = c6 * (3 * x * x - y * y - 3 * z * z)
        g[..., 15, 1], g[..., 15, 2] = c6 * (-2 * x * y), c6 * (-6 * x * z)
    return g


# ---------------------------------------------------------------- preprocess
def prepare(model, cam, light, subset=None, cutoff=True):
    """Per visible Gaussian, in row order (ref render.py:226-290).

    ``light`` = dict(direction (3,), intensity (3,), ambient (3,BL) or None),
    direction already normalised.  Returns a dict of arrays.
    """
    rows = np.arange(model.means.shape[0]) if subset is None else np.sort(np.asarray(subset, np.int64))
    P = np.asarray(model.means, np.float64)[rows]
    Rc = cam["R"]
    d = P - cam["pos"]
    mc = np.stack([(d[:, 0] * Rc[0, k] + d[:, 1] * Rc[1, k]) + d[:, 2] * Rc[2, k] for k in range(3)], -1)
    vis = mc[:, 2] >= cam["near"]
    rows, P, d, mc = rows[vis], P[vis], d[vis], mc[vis]
    M = rows.size
    ls = np.asarray(model.log_scales, np.float64)[rows]
    q = np.asarray(model.quaternions, np.float64)[rows]
    sh = np.asarray(model.sh_coeffs, np.float64)[rows]
    logit = np.asarray(model.logit_opacities, np.float64)[rows]
    lvis = np.asarray(model.light_visibility, np.float64)[rows]
    degree = int(model.sh_degree)

    x, y, z = mc[:, 0], mc[:, 1], mc[:, 2]
    fx, fy = cam["fx"], cam["fy"]
    J = np.zeros((M, 2, 3))
    J[:, 0, 0] = fx / z
    J[:, 0, 2] = (-fx * x) / (z * z)
    J[:, 1, 1] = fy / z
    J[:, 1, 2] = (-fy * y) / (z * z)
    mu2d = np.stack([(fx * x) / z + cam["cx"], (fy * y) / z + cam["cy"]], -1)

    Rq = quat_rotmat(q)
    S2 = det_exp(2.0 * ls)
    S3 = np.empty((M, 3, 3))
    for i in range(3):
        for j in range(3):
            S3[:, i, j] = ((Rq[:, i, 0] * S2[:, 0]) * Rq[:, j, 0]
                           + (Rq[:, i, 1] * S2[:, 1]) * Rq[:, j, 1]) + (Rq[:, i, 2] * S2[:, 2]) * Rq[:, j, 2]
    Wm = Rc.T
    Tm = np.empty((M, 3, 3))
    for i in range(3):
        for l in range(3):
            Tm[:, i, l] = (Wm[i, 0] * S3[:, 0, l] + Wm[i, 1] * S3[:, 1, l]) + Wm[i, 2] * S3[:, 2, l]
    cov = np.empty((M, 3, 3))
    for i in range(3):
        for j in range(3):
            cov[:, i, j] = (Tm[:, i, 0] * Wm[j, 0] + Tm[:, i, 1] * Wm[j, 1]) + Tm[:, i, 2] * Wm[j, 2]
    U0 = [J[:, 0, 0] * cov[:, 0, l] + J[:, 0, 2] * cov[:, 2, l] for l in range(3)]
    U1 = [J[:, 1, 1] * cov[:, 1, l] + J[:, 1, 2] * cov[:, 2, l] for l in range(3)]
    s00 = (U0[0] * J[:, 0, 0] + U0[2] * J[:, 0, 2]) + BLUR
    s01 = U0[1] * J[:, 1, 1] + U0[2] * J[:, 1, 2]
    s11 = (U1[1] * J[:, 1, 1] + U1[2] * J[:, 1, 2]) + BLUR
    det = s00 * s11 - s01 * s01
    Sig2 = np.stack([np.stack([s00, s01], -1), np.stack([s01, s11], -1)], -2)
    inv2 = np.stack([np.stack([s11 / det, -s01 / det], -1), np.stack([-s01 / det, s00 / det], -1)], -2)

    if cutoff:
        tr = s00 + s11
        lam = 0.5 * tr + np.sqrt(np.maximum(0.25 * (tr * tr) - det, 0.0))
        radius = 3.0 * np.sqrt(lam)
    else:
        radius = np.full(M, np.inf)
    rect = windows(mu2d, radius, cam["W"], cam["H"])

    # appearance (ref render.py:175-197 with the normal proxy of render.py:139-151)
    dist = np.sqrt(((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]))
    vdir = d / dist[:, None]
    k = np.argmax(ls <= ls.min(axis=1, keepdims=True) + AXIS_MARGIN, axis=1) if M else np.zeros(0, np.int64)
    n_hat = Rq[np.arange(M), :, k]
    Y = sh_basis(vdir, degree)
    ldir = np.asarray(light["direction"], np.float64)
    inten = np.asarray(light["intensity"], np.float64)
    s = n_hat @ (-ldir)
    cosv = np.abs(s)
    albedo = SH_C0 * sh[:, :, 0] + 0.5
    direct = albedo * inten[None, :] * (cosv * lvis)[:, None]
    amb = light.get("ambient")
    if amb is None:
        base = (sh * Y[:, None, :]).sum(-1) + 0.5
    else:
        amb = np.asarray(amb, np.float64)
        BL = min(amb.shape[1], sh.shape[2])
        eff = sh[:, :, :BL].copy()
        eff[:, :, 0] += 0.5 / SH_C0
        base = (eff * amb[None, :, :BL]).sum(-1)
        if sh.shape[2] > 1:
            base = base + (sh[:, :, 1:] * Y[:, None, 1:]).sum(-1)
    color_pre = base + direct
    color = np.clip(color_pre, 0.0, 1.0)
    opacity = 1.0 / (1.0 + np.exp(-logit))

    key = mc[:, 2].view(np.uint64) if M else np.zeros(0, np.uint64)
    order = np.argsort(key, kind="stable")  # rows ascending -> ties by row
    return dict(rows=rows, mu_cam=mc, depth=mc[:, 2], mu2d=mu2d, J=J, Rq=Rq, S2=S2, Sigma3d=S3,
                cov_cam=cov, Sigma2d=Sig2, inv2d=inv2, det=det, radius=radius, rect=rect,
                opacity=opacity, color=color, color_pre=color_pre, view_dir=vdir, view_dist=dist,
                n_hat=n_hat, n_axis=k, s=s, cos=cosv, Y=Y, albedo=albedo, lvis=lvis, sh=sh,
                ls=ls, quat=q, order=order, degree=degree)


def windows(mu2d, radius, W, H):
    """(M,4) int64 [x0, x1, y0, y1) (ref render.py:293-301)."""
    M = mu2d.shape[0]
    out = np.empty((M, 4), np.int64)
    inf = ~np.isfinite(radius)
    with np.errstate(invalid="ignore"):
        lo_x = np.floor(mu2d[:, 0] - radius)
        hi_x = np.ceil(mu2d[:, 0] + radius) + 1
        lo_y = np.floor(mu2d[:, 1] - radius)
        hi_y = np.ceil(mu2d[:, 1] + radius) + 1
    out[:, 0] = np.clip(np.where(inf, 0, lo_x), 0, W)
    out[:, 1] = np.clip(np.where(inf, W, hi_x), 0, W)
    out[:, 2] = np.clip(np.where(inf, 0, lo_y), 0, H)
    out[:, 3] = np.clip(np.where(inf, H, hi_y), 0, H)
    # a window clipped to the far side of the image is empty either way
    out[:, 0] = np.minimum(out[:, 0], W)
    out[:, 2] = np.minimum(out[:, 2], H)
    return out


def tile_bins(prep, W, H, tile=TILE):
    """Depth-ordered rows and per-tile splat lists (the GPU's K2-K4 products).

    Returns dict(order_rows, ranges (T,2) int64, pair_rank (P,) int64, tile_count (M_sorted,)).
    A splat of depth rank r touches tile (tx,ty) iff its window intersects it.
    """
    tw, th = -(-W // tile), -(-H // tile)
    rect = prep["rect"][prep["order"]]
    nonempty = (rect[:, 0] < rect[:, 1]) & (rect[:, 2] < rect[:, 3])
    tiles, ranks = [], []
    for r in np.flatnonzero(nonempty):
        x0, x1, y0, y1 = rect[r]
        tx = np.arange(x0 // tile, (x1 - 1) // tile + 1)
        ty = np.arange(y0 // tile, (y1 - 1) // tile + 1)
        t = (ty[:, None] * tw + tx[None, :]).ravel()
        tiles.append(t)
        ranks.append(np.full(t.size, r))
    tiles = np.concatenate(tiles) if tiles else np.zeros(0, np.int64)
    ranks = np.concatenate(ranks) if ranks else np.zeros(0, np.int64)
    o = np.lexsort((ranks, tiles))
    tiles, ranks = tiles[o], ranks[o]
    ranges = np.zeros((tw * th, 2), np.int64)
    bounds = np.searchsorted(tiles, np.arange(tw * th + 1))
    ranges[:, 0], ranges[:, 1] = bounds[:-1], bounds[1:]
    return dict(order_rows=prep["rows"][prep["order"]], ranges=ranges, pair_rank=ranks, pair_tile=tiles)


# ---------------------------------------------------------------- blending
def _alpha(prep, i, x0, x1, y0, y1):
    dx = (np.arange(x0, x1, dtype=np.float64) + 0.5)[None, :] - prep["mu2d"][i, 0]
    dy = (np.arange(y0, y1, dtype=np.float64) + 0.5)[:, None] - prep["mu2d"][i, 1]
    A = prep["inv2d"][i]
    power = -0.5 * (A[0, 0] * dx * dx + 2.0 * A[0, 1] * dx * dy + A[1, 1] * dy * dy)
    G = np.exp(power)
    return np.minimum(prep["opacity"][i] * G, ALPHA_CAP), G, dx, dy


def _clip(rect, crop):
    """The window [x0,x1)x[y0,y1) restricted to crop (cx0, cx1, cy0, cy1): (absolute
    x0, x1, y0, y1, and the same relative to the crop origin)."""
    x0, x1, y0, y1 = rect
    cx0, cx1, cy0, cy1 = crop
    x0, x1, y0, y1 = max(x0, cx0), min(x1, cx1), max(y0, cy0), min(y1, cy1)
    return (x0, x1, y0, y1), (x0 - cx0, x1 - cx0, y0 - cy0, y1 - cy0)


def composite(prep, W, H, bg, crop=None):
    """Front-to-back compositing in depth order (ref render.py:317-336).
    Returns (image (H,W,3), T (H,W), pairs) where pairs counts the
    (pixel, splat) evaluations that passed the T-gate.  With crop =
    (x0, x1, y0, y1) only those pixels of the (W, H) frame are composited
    (per-pixel results identical to the full frame's: every splat whose
    window meets the crop is walked, in the same order)."""
    crop = (0, W, 0, H) if crop is None else tuple(int(v) for v in crop)
    h, w_ = crop[3] - crop[2], crop[1] - crop[0]
    img = np.zeros((h, w_, 3))
    T = np.ones((h, w_))
    pairs = 0
    for i in prep["order"]:
        (x0, x1, y0, y1), (a0, a1, b0, b1) = _clip(prep["rect"][i], crop)
        if x0 >= x1 or y0 >= y1:
            continue
        Tw = T[b0:b1, a0:a1]
        live = Tw >= T_CUTOFF
        n_live = int(live.sum())
        if n_live == 0:
            continue
        pairs += n_live
        a, _, _, _ = _alpha(prep, i, x0, x1, y0, y1)
        w = np.where(live, a * Tw, 0.0)
        img[b0:b1, a0:a1] += w[..., None] * prep["color"][i]
        T[b0:b1, a0:a1] = np.where(live, Tw * (1.0 - a), Tw)
    img += T[..., None] * np.asarray(bg, np.float64)
    return img, T, pairs


def screen_grads(prep, image, gt, W, H, crop=None):
    """The per-splat front-to-back walk of ref optim.py:133-172.
    Returns (g_color (M,3), g_opacity (M,), g_mu2d (M,2), g_sig (M,3) = [00,01,11]).
    With crop, image / gt are the crop's pixels of the (W, H) frame and the
    sums run over them only (complete for splats whose window lies inside the
    crop); dL/dC keeps the full frame's normalisation 1/(H*W*3)."""
    crop = (0, W, 0, H) if crop is None else tuple(int(v) for v in crop)
    M = prep["rows"].size
    dLdC = np.sign(image - gt) / (H * W * 3)
    gc = np.zeros((M, 3))
    go = np.zeros(M)
    gm = np.zeros((M, 2))
    gs = np.zeros((M, 3))
    T = np.ones(image.shape[:2])
    prefix = np.zeros(image.shape)
    for i in prep["order"]:
        (x0, x1, y0, y1), (a0, a1, b0, b1) = _clip(prep["rect"][i], crop)
        if x0 >= x1 or y0 >= y1:
            continue
        Tw = T[b0:b1, a0:a1]
        live = Tw >= T_CUTOFF
        if not live.any():
            continue
        a, G, dx, dy = _alpha(prep, i, x0, x1, y0, y1)
        open_ = prep["opacity"][i] * G < ALPHA_CAP
        w = np.where(live, a * Tw, 0.0)
        g = dLdC[b0:b1, a0:a1]
        col = prep["color"][i]
        gc[i] = (g * w[..., None]).sum(axis=(0, 1))
        S = image[b0:b1, a0:a1] - prefix[b0:b1, a0:a1] - w[..., None] * col
        da = (g * (col[None, None, :] * Tw[..., None] - S / (1.0 - a)[..., None])).sum(-1)
        da = np.where(live, da, 0.0)
        go[i] = (da * np.where(open_, G, 0.0)).sum()
        gp = da * np.where(open_, a, 0.0)
        A = prep["inv2d"][i]
        ax = A[0, 0] * dx + A[0, 1] * dy
        ay = A[1, 0] * dx + A[1, 1] * dy
        gm[i] = [(gp * ax).sum(), (gp * ay).sum()]
        gs[i] = [0.5 * (gp * ax * ax).sum(), 0.5 * (gp * ax * ay).sum(), 0.5 * (gp * ay * ay).sum()]
        prefix[b0:b1, a0:a1] += w[..., None] * col
        T[b0:b1, a0:a1] = np.where(live, Tw * (1.0 - a), Tw)
    return gc, go, gm, gs


def chain_rule(prep, cam, light, gc, go, gm, gs):
    """Per-Gaussian parameter gradients from the screen-space ones (ref optim.py:174-244)."""
    M = prep["rows"].size
    pre = prep["color_pre"]
    gc = np.where((pre > 0.0) & (pre < 1.0), gc, 0.0)
    G2 = np.zeros((M, 2, 2))
    G2[:, 0, 0], G2[:, 0, 1], G2[:, 1, 0], G2[:, 1, 1] = gs[:, 0], gs[:, 1], gs[:, 1], gs[:, 2]
    J, cov = prep["J"], prep["cov_cam"]
    gJ = 2.0 * G2 @ J @ cov                              # (G2 + G2^T) J cov
    gV = np.swapaxes(J, 1, 2) @ G2 @ J                   # J^T G2 J
    Wm = cam["R"].T
    G3 = Wm.T[None] @ gV @ Wm[None]                      # W^T gV W
    fx, fy = cam["fx"], cam["fy"]
    x, y, z = prep["mu_cam"].T
    gmc = (np.swapaxes(J, 1, 2) @ gm[:, :, None])[:, :, 0]
    gmc[:, 0] += gJ[:, 0, 2] * (-fx / z ** 2)
    gmc[:, 1] += gJ[:, 1, 2] * (-fy / z ** 2)
    gmc[:, 2] += (gJ[:, 0, 0] * (-fx / z ** 2) + gJ[:, 1, 1] * (-fy / z ** 2)
                  + gJ[:, 0, 2] * (2 * fx * x / z ** 3) + gJ[:, 1, 2] * (2 * fy * y / z ** 3))
    g_mean = gmc @ Wm

    Rq, S2 = prep["Rq"], prep["S2"]
    RtGR = np.swapaxes(Rq, 1, 2) @ G3 @ Rq
    g_ls = np.diagonal(RtGR, axis1=1, axis2=2) * 2.0 * S2
    gR = ((G3 + np.swapaxes(G3, 1, 2)) @ Rq) * S2[:, None, :]
    inten = np.asarray(light["intensity"], np.float64)
    toward = -np.asarray(light["direction"], np.float64)
    g_cos = (gc * prep["albedo"] * inten[None, :]).sum(-1) * prep["lvis"]
    g_s = g_cos * np.sign(prep["s"])
    gR[np.arange(M), :, prep["n_axis"]] += g_s[:, None] * toward[None, :]
    g_quat = (gR[:, None, :, :] * drot_dquat(prep["quat"])).sum(axis=(2, 3))

    sh, Y = prep["sh"], prep["Y"]
    B = sh.shape[2]
    g_sh = np.zeros((M, 3, B))
    amb = light.get("ambient")
    if amb is None:
        g_sh += gc[:, :, None] * Y[:, None, :]
    else:
        amb = np.asarray(amb, np.float64)
        BL = min(amb.shape[1], B)
        g_sh[:, :, :BL] += gc[:, :, None] * amb[None, :, :BL]
        if B > 1:
            g_sh[:, :, 1:] += gc[:, :, None] * Y[:, None, 1:]
    g_sh[:, :, 0] += gc * (SH_C0 * inten[None, :]) * (prep["cos"] * prep["lvis"])[:, None]

    dY = sh_basis_jac(prep["view_dir"], prep["degree"])
    g_v = np.einsum("mcb,mc,mbk->mk", sh, gc, dY)
    v = prep["view_dir"]
    proj = (np.eye(3)[None] - v[:, :, None] * v[:, None, :]) / prep["view_dist"][:, None, None]
    g_mean = g_mean + (proj @ g_v[:, :, None])[:, :, 0]
    op = prep["opacity"]
    g_logit = go * op * (1.0 - op)
    return dict(means=g_mean, log_scales=g_ls, quaternions=g_quat, logit_opacities=g_logit, sh_coeffs=g_sh)


def backward(model, cam, light, gt, bg=(0.0, 0.0, 0.0), subset=None, cutoff=True):
    """(loss, grads over active rows (dict of f64 arrays), image).  ref optim.py:113-268."""
    prep = prepare(model, cam, light, subset, cutoff)
    W, H = cam["W"], cam["H"]
    img, _, _ = composite(prep, W, H, bg)
    gt = np.asarray(gt, np.float64)
    L = float(np.mean(np.abs(img - gt)))
    gc, go, gm, gs = screen_grads(prep, img, gt, W, H)
    per = chain_rule(prep, cam, light, gc, go, gm, gs)
    n = model.means.shape[0]
    a = int(model.active_count)
    B = np.asarray(model.sh_coeffs).shape[2]
    shapes = dict(means=(n, 3), log_scales=(n, 3), quaternions=(n, 4), logit_opacities=(n,), sh_coeffs=(n, 3, B))
    grads = {}
    for name, shp in shapes.items():
        full = np.zeros(shp)
        full[prep["rows"]] = per[name]
        grads[name] = full[:a]
    return L, grads, img


def render(model, cam, light, bg=(0.0, 0.0, 0.0), subset=None, cutoff=True):
    prep = prepare(model, cam, light, subset, cutoff)
    img, T, _ = composite(prep, cam["W"], cam["H"], bg)
    return img, T
