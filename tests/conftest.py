"""Shared fixtures: golden-vector loading and the gpu marker.

`-m "not gpu"` runs here (no GPU): the oracle against the reference's golden
vectors, host logic, gloo multi-process tests, and the C-ABI load check.
`-m gpu` runs on a B200: CUDA path vs oracle/golden through the C ABI.
"""

import json
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


class Case(dict):
    """Golden case: metadata keys plus lazily loaded arrays via .a(name)."""

    def __init__(self, meta, npz):
        super().__init__(meta)
        self._npz = npz

    def a(self, name):
        return self._npz[f"c{self['id']}_{name}"]

    def has(self, name):
        return name in self["arrays"]


_CACHE = {}


def load_cases(stem):
    if stem not in _CACHE:
        meta = json.loads((GOLDEN / f"{stem}.json").read_text())
        npz = np.load(GOLDEN / f"{stem}.npz")
        _CACHE[stem] = [Case(m, npz) for m in meta]
    return _CACHE[stem]


class NS:
    """Attribute bag used to hand arrays to the oracle / product APIs."""

    def __init__(self, **kw):
        self.__dict__.update(kw)


def case_model(c, prefix=""):
    g = lambda k: np.array(c.a(prefix + k))
    sh = g("sh_coeffs")
    return NS(means=g("means"), log_scales=g("log_scales"), quaternions=g("quaternions"),
              logit_opacities=g("logit_opacities"), sh_coeffs=sh, light_visibility=g("light_visibility"),
              object_ids=g("object_ids"), active_count=int(c["active"]),
              sh_degree=int(round(np.sqrt(sh.shape[2]))) - 1)


@pytest.fixture
def golden():
    return load_cases
