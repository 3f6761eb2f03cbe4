"""Alias conftest: the reference's own tests against the B200 drop-in.

Installed as baseline/_ref_tests/tests/conftest.py by tests/refsuite/prepare.py
next to UNMODIFIED copies of the reference's test files (SURVEY §4 reuse
plan).  Before any test module imports them, the hot-path entry points of
the reference package (`splatstream`, installed in baseline/_ref) are
replaced by the drop-in's, in their fp64 blend instantiation (SURVEY
Appendix B: the reference tests hold fp64-level tolerances):

  splatstream.render    render, prepare_splats, composite, update_light_visibility
  splatstream.optim     backward, step, OptimizerState
  splatstream.protocol  encode_delta, encode_snapshot, decode_snapshot, decode_delta,
                        apply_delta, advance_baseline

The reference's StreamServer / StreamClient (test_server.py, test_client.py)
import those names, so their whole tick loop -- optimizer step, snapshot,
delta emission, client ingestion -- runs on the drop-in.

Everything else (geometry, model, scene, engine, the numpy helpers
shade_gaussian / sh_basis / normal_proxies / _drotmat_dquat_batch, framing,
packets) stays the reference's -- those are not on the hot path (SURVEY
Appendix B, last row).  Exclusions are listed in tests/test_gpu_reference_suite.py.
"""

import functools
import os
import sys

ROOT = os.environ.get("SS_REPO_ROOT")
if ROOT and ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import splatstream.optim as _O  # noqa: E402
import splatstream.protocol as _P  # noqa: E402
import splatstream.protocol.delta as _PD  # noqa: E402
import splatstream.protocol.snapshot as _PS  # noqa: E402
import splatstream.render as _R  # noqa: E402

from paper_2604_02851_b200 import optim as _o2  # noqa: E402
from paper_2604_02851_b200 import protocol as _p2  # noqa: E402
from paper_2604_02851_b200 import render as _r2  # noqa: E402
from paper_2604_02851_b200.protocol import ingest as _i2  # noqa: E402


def _fp64(fn):
    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        kwargs.setdefault("precision", 1)
        return fn(*args, **kwargs)
    return wrapped


def _decode_snapshot(payload):
    """The drop-in's device decode, returned as the caller's own host model
    type (the reference's GaussianModel, whose mutation methods the client
    uses on its replica)."""
    import splatstream.model as _M
    m, info = _i2.decode_snapshot_host(payload)
    return _M.GaussianModel(means=m.means, log_scales=m.log_scales, quaternions=m.quaternions,
                            logit_opacities=m.logit_opacities, sh_coeffs=m.sh_coeffs,
                            light_visibility=m.light_visibility, object_ids=m.object_ids,
                            active_count=m.active_count, sh_degree=m.sh_degree), info


_PATCH = {
    _R: dict(render=_fp64(_r2.render), prepare_splats=_r2.prepare_splats, composite=_r2.composite,
             update_light_visibility=_r2.update_light_visibility),
    _O: dict(backward=_fp64(_o2.backward), step=_fp64(_o2.step), OptimizerState=_o2.OptimizerState),
    _P: dict(encode_delta=_p2.encode_delta, encode_snapshot=_p2.encode_snapshot,
             decode_snapshot=_decode_snapshot, decode_delta=_i2.decode_delta_host,
             apply_delta=_i2.apply_delta),
    _PD: dict(encode_delta=_p2.encode_delta, decode_delta=_i2.decode_delta_host, apply_delta=_i2.apply_delta,
              advance_baseline=_i2.advance_baseline),
    _PS: dict(encode_snapshot=_p2.encode_snapshot, decode_snapshot=_decode_snapshot),
}
for _mod, _names in _PATCH.items():
    for _k, _v in _names.items():
        setattr(_mod, _k, _v)

# one ProtocolError: the drop-in raises the reference's exception class, so
# `pytest.raises(splatstream.protocol.ProtocolError)` catches it
from paper_2604_02851_b200 import errors as _errors  # noqa: E402
from splatstream.protocol.framing import ProtocolError as _RefProtocolError  # noqa: E402

_ours = _errors.ProtocolError
for _name, _m in list(sys.modules.items()):
    if _name.startswith("paper_2604_02851_b200") and getattr(_m, "ProtocolError", None) is _ours:
        _m.ProtocolError = _RefProtocolError
