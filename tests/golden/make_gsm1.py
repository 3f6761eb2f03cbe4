"""Golden GSM1 containers written by the unmodified reference's save_model
(ref pkg/src/splatstream/model.py:410-416).  Run in the build container:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_gsm1.py
Writes tests/golden/gsm1_deg{1,3}.bin and gsm1_cases.npz (the inputs)."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from splatstream.model import GaussianModel, save_model  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(7)
arrays = {}
for deg, n, a in ((1, 37, 30), (3, 101, 64)):
    B = (deg + 1) ** 2
    m = GaussianModel(means=rng.normal(size=(n, 3)).astype(np.float32),
                      log_scales=rng.normal(-3, 1, (n, 3)).astype(np.float32),
                      quaternions=rng.normal(size=(n, 4)).astype(np.float32),
                      logit_opacities=rng.normal(size=n).astype(np.float32),
                      sh_coeffs=rng.normal(size=(n, 3, B)).astype(np.float32),
                      light_visibility=rng.random(n).astype(np.float32),
                      object_ids=rng.integers(-1, 5, n).astype(np.int32),
                      active_count=a, sh_degree=deg)
    save_model(os.path.join(HERE, f"gsm1_deg{deg}.bin"), m)
    for k in ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs", "light_visibility", "object_ids"):
        arrays[f"deg{deg}_{k}"] = getattr(m, k)
    arrays[f"deg{deg}_meta"] = np.array([n, a, deg])
np.savez(os.path.join(HERE, "gsm1_cases.npz"), **arrays)
print("ok")
