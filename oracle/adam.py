"""CPU restatement of the optimizer step (test infrastructure only).

ref pkg/src/splatstream/optim.py:281-407 (OptimizerState, step): the per-view
gradients are summed, scaled by 1/len(views), and applied with bias-corrected
Adam whose moments are float64; the parameter update is computed in float64
and stored as float32; quaternions are renormalised; the per-row grad-norm
EMA (fresh rows take the norm directly) and age are advanced.
"""

from __future__ import annotations

import numpy as np

GROUPS = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs")


class AdamState:
    def __init__(self, a, B, lrs=None, scene_extent=1.0, betas=(0.9, 0.999), eps=1e-8, ema_beta=0.99):
        self.lrs = dict(means=2e-4, log_scales=5e-3, quaternions=1e-3, logit_opacities=5e-2,
                        sh_dc=2.5e-3, sh_rest=1.25e-4)
        if lrs:
            self.lrs.update(lrs)
        self.scene_extent = float(scene_extent)
        self.betas, self.eps, self.ema_beta = betas, eps, ema_beta
        shapes = dict(means=(a, 3), log_scales=(a, 3), quaternions=(a, 4), logit_opacities=(a,),
                      sh_coeffs=(a, 3, B))
        self.m = {k: np.zeros(s) for k, s in shapes.items()}
        self.v = {k: np.zeros(s) for k, s in shapes.items()}
        self.age = np.zeros(a, np.int64)
        self.grad_ema = np.zeros(a)
        self.step_count = 0


def apply(model, state: AdamState, grads_sum: dict, n_views: int):
    """Adam on model[:a] in place from summed per-view grads (dict of f64)."""
    a = int(model.active_count)
    if a == 0:
        return
    g = {k: np.asarray(v, np.float64) * (1.0 / n_views) for k, v in grads_sum.items()}
    state.step_count += 1
    t = state.step_count
    b1, b2 = state.betas
    for k in GROUPS:
        state.m[k] = b1 * state.m[k] + (1 - b1) * g[k]
        state.v[k] = b2 * state.v[k] + (1 - b2) * g[k] * g[k]
        upd = (state.m[k] / (1 - b1 ** t)) / (np.sqrt(state.v[k] / (1 - b2 ** t)) + state.eps)
        if k == "sh_coeffs":
            upd[:, :, 0] *= state.lrs["sh_dc"]
            upd[:, :, 1:] *= state.lrs["sh_rest"]
        elif k == "means":
            upd *= state.lrs["means"] * state.scene_extent
        else:
            upd *= state.lrs[k]
        arr = getattr(model, k)
        arr[:a] = (arr[:a].astype(np.float64) - upd).astype(np.float32)
    q = model.quaternions[:a].astype(np.float64)
    n = np.sqrt(((q[:, 0] * q[:, 0] + q[:, 1] * q[:, 1]) + q[:, 2] * q[:, 2]) + q[:, 3] * q[:, 3])
    model.quaternions[:a] = (q / n[:, None]).astype(np.float32)
    gm = g["means"]
    norms = np.sqrt(((gm[:, 0] * gm[:, 0] + gm[:, 1] * gm[:, 1]) + gm[:, 2] * gm[:, 2]))
    fresh = state.age == 0
    state.grad_ema = np.where(fresh, norms, state.ema_beta * state.grad_ema + (1 - state.ema_beta) * norms)
    state.age += 1
