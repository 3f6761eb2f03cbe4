"""Gaussian stores: the reference's host layout and its HBM-resident twin.

GaussianModel   host numpy columns, same fields and layout as ref
                pkg/src/splatstream/model.py:233-298 (active rows first).
DeviceModel     the same columns as contiguous torch CUDA tensors -- the
                layout the kernels read (SoA per attribute, float32, AoS
                within an attribute exactly like the numpy arrays), so one
                ss_model struct of pointers describes it.  At 1M rows and SH
                degree 3 it is 244 MB of HBM.

Every entry point accepts either: a host model is uploaded for the call
(and trainable rows are written back where the reference mutates in place);
a DeviceModel stays resident.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

ATTRIBUTE_NAMES = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs",
                   "light_visibility", "object_ids")
TRAINABLE = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs")


def num_sh_bases(degree: int) -> int:
    return (degree + 1) ** 2


@dataclass
class GaussianModel:
    means: np.ndarray
    log_scales: np.ndarray
    quaternions: np.ndarray
    logit_opacities: np.ndarray
    sh_coeffs: np.ndarray
    light_visibility: np.ndarray
    object_ids: np.ndarray
    active_count: int
    sh_degree: int

    @property
    def count(self) -> int:
        return self.means.shape[0]

    @staticmethod
    def empty(sh_degree: int = 0) -> "GaussianModel":
        B = num_sh_bases(sh_degree)
        z = np.zeros
        return GaussianModel(z((0, 3), np.float32), z((0, 3), np.float32), z((0, 4), np.float32),
                             z(0, np.float32), z((0, 3, B), np.float32), z(0, np.float32), z(0, np.int32),
                             0, sh_degree)

    def copy(self) -> "GaussianModel":
        return GaussianModel(*(getattr(self, k).copy() for k in ATTRIBUTE_NAMES), self.active_count, self.sh_degree)

    def attribute(self, name: str):
        return getattr(self, name)


class DeviceModel:
    """HBM-resident columns (torch CUDA tensors) with the reference's field names."""

    def __init__(self, means, log_scales, quaternions, logit_opacities, sh_coeffs, light_visibility, object_ids,
                 active_count: int, sh_degree: int):
        self.means = means
        self.log_scales = log_scales
        self.quaternions = quaternions
        self.logit_opacities = logit_opacities
        self.sh_coeffs = sh_coeffs
        self.light_visibility = light_visibility
        self.object_ids = object_ids
        self.active_count = int(active_count)
        self.sh_degree = int(sh_degree)

    @property
    def count(self) -> int:
        return int(self.means.shape[0])

    @property
    def device(self):
        return self.means.device

    def attribute(self, name: str):
        return getattr(self, name)

    @staticmethod
    def from_host(model, device=None, keep_f64: bool = False) -> "DeviceModel":
        """Upload a host model: float32 columns, or -- with keep_f64 and a
        model whose means are float64 (the reference's unit tests build such
        models) -- float64 columns for the fp64 blend instantiation, so a
        finite-difference perturbation of 1e-4 reaches the kernels intact."""
        import torch
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        f64 = keep_f64 and np.asarray(model.means).dtype == np.float64
        ft = np.float64 if f64 else np.float32

        def up(a, dt):
            return torch.from_numpy(np.ascontiguousarray(np.asarray(a), dtype=dt)).to(dev, non_blocking=False)

        return DeviceModel(up(model.means, ft).reshape(-1, 3), up(model.log_scales, ft).reshape(-1, 3),
                           up(model.quaternions, ft).reshape(-1, 4),
                           up(model.logit_opacities, ft).reshape(-1),
                           up(model.sh_coeffs, ft), up(model.light_visibility, ft).reshape(-1),
                           up(model.object_ids, np.int32).reshape(-1), model.active_count, model.sh_degree)

    def to_host(self) -> GaussianModel:
        return GaussianModel(*(getattr(self, k).cpu().numpy() for k in ATTRIBUTE_NAMES), self.active_count,
                             self.sh_degree)

    def write_back(self, model, names=TRAINABLE, rows=None):
        """Copy device columns into a host model in place (rows [0, rows))."""
        n = self.count if rows is None else rows
        for k in names:
            dst = getattr(model, k)
            src = getattr(self, k)[:n].cpu().numpy()
            dst[:n] = src.astype(dst.dtype, copy=False).reshape(dst[:n].shape)

    def struct(self) -> _lib.SSModel:
        s = _lib.SSModel()
        for k in ATTRIBUTE_NAMES:
            t = getattr(self, k)
            assert t.is_cuda and t.is_contiguous(), k
            setattr(s, k, t.data_ptr())
        s.count = self.count
        s.active_count = self.active_count
        s.sh_degree = self.sh_degree
        s.param_dtype = 1 if self.means.dtype == torch_float64() else 0
        return s

    def clone(self) -> "DeviceModel":
        return DeviceModel(*(getattr(self, k).clone() for k in ATTRIBUTE_NAMES), self.active_count, self.sh_degree)


def torch_float64():
    import torch
    return torch.float64


def as_device(model, device=None, keep_f64: bool = False):
    """(DeviceModel, uploaded?) for either kind of model (keep_f64: see
    DeviceModel.from_host; only the fp64 blend entry points pass it)."""
    if isinstance(model, DeviceModel):
        return model, False
    return DeviceModel.from_host(model, device, keep_f64), True


# ---------------------------------------------------------------- GSM1 container (ref model.py:407-442)
MODEL_MAGIC = b"GSM1"


def save_model(path, model) -> None:
    """ref model.py:410-416: magic, <III (sh_degree, count, active_count), then
    every attribute as little-endian float32 (object ids too), in
    ATTRIBUTE_NAMES order.  A DeviceModel is read back attribute by
    attribute; the bytes equal the reference's for the same rows."""
    import struct
    with open(path, "wb") as f:
        f.write(MODEL_MAGIC)
        f.write(struct.pack("<III", model.sh_degree, model.count, model.active_count))
        for name in ATTRIBUTE_NAMES:
            a = getattr(model, name)
            if not isinstance(a, np.ndarray):  # a CUDA tensor of a DeviceModel
                a = a.cpu().numpy()
            f.write(np.ascontiguousarray(a, dtype="<f4").tobytes())


def load_model(path, device=None):
    """ref model.py:419-442: the container as a host GaussianModel, or, with
    `device`, uploaded as a DeviceModel."""
    import struct
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] != MODEL_MAGIC:
        raise ValueError("not a model container")
    sh_degree, count, active_count = struct.unpack_from("<III", data, 4)
    B = num_sh_bases(sh_degree)
    shapes = {"means": (count, 3), "log_scales": (count, 3), "quaternions": (count, 4), "logit_opacities": (count,),
              "sh_coeffs": (count, 3, B), "light_visibility": (count,), "object_ids": (count,)}
    off = 16
    arrays = {}
    for name in ATTRIBUTE_NAMES:
        n = int(np.prod(shapes[name]))
        arr = np.frombuffer(data, dtype="<f4", count=n, offset=off).reshape(shapes[name])
        off += 4 * n
        arrays[name] = arr.astype(np.int32) if name == "object_ids" else arr.astype(np.float32)
    host = GaussianModel(active_count=active_count, sh_degree=sh_degree, **arrays)
    if device is None:
        return host
    return DeviceModel.from_host(host, device)
