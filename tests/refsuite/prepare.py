#!/usr/bin/env python3
"""Stage the reference's own hot-path test suites for a run against the drop-in.

Copies, UNMODIFIED, the reference's pkg/tests/{test_render, test_optim,
test_protocol, test_golden}.py, its golden-packet script and manifest, plus
the regenerated wire fixtures (tests/golden/wire, produced by that script)
into baseline/_ref_tests/ (git-ignored, like the reference install in
baseline/_ref; both travel to the GPU box), and installs
tests/refsuite/alias_conftest.py there as the suite's conftest.py.

Runs where /root/reference exists (this build container; __graft_entry__.build()
calls it).  tests/test_gpu_reference_suite.py runs the staged suite on the GPU.
"""

from __future__ import annotations

import pathlib
import shutil
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
REF = pathlib.Path("/root/reference/pkg")
OUT = ROOT / "baseline" / "_ref_tests"
SUITES = ("test_render.py", "test_optim.py", "test_protocol.py", "test_golden.py", "test_server.py", "test_client.py")


def prepare(ref: pathlib.Path = REF) -> bool:
    if not (ref / "tests").is_dir():
        return False
    if OUT.exists():
        shutil.rmtree(OUT)
    (OUT / "tests" / "golden").mkdir(parents=True)
    (OUT / "scripts").mkdir()
    for name in SUITES:
        shutil.copy2(ref / "tests" / name, OUT / "tests" / name)
    shutil.copy2(ref / "scripts" / "make_golden_packets.py", OUT / "scripts" / "make_golden_packets.py")
    for f in (ROOT / "tests" / "golden" / "wire").iterdir():
        shutil.copy2(f, OUT / "tests" / "golden" / f.name)
    shutil.copy2(ROOT / "tests" / "refsuite" / "alias_conftest.py", OUT / "tests" / "conftest.py")
    return True


if __name__ == "__main__":
    ok = prepare(pathlib.Path(sys.argv[1]) if len(sys.argv) > 1 else REF)
    print("staged" if ok else "reference tests not found", OUT)
