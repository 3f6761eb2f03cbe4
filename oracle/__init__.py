"""CPU oracle for the splatstream hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, on the CPU, the reference algorithms that the B200
kernels in ``paper_2604_02851_b200`` replace.  It exists so that the parity
tests (``tests/``), ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` have an independent checker.  The
product package never imports it; the product fails loudly when its CUDA
library is missing instead of falling back here.

Pinning: every module is checked against golden vectors produced by the
unmodified reference (``/root/reference/pkg``) with the committed generator
``tests/golden/make_golden.py`` -- the wire fixtures of
``pkg/scripts/make_golden_packets.py`` plus encoder, renderer, backward and
optimizer vectors.  See ``tests/test_oracle_golden.py``.

Modules
  codec     quantizers, bit packing, varints, delta + snapshot encoders
            (ref pkg/src/splatstream/protocol/{quantize,delta,snapshot}.py)
  raster    fp64 preprocess, window/tile binning, composite, backward
            (ref pkg/src/splatstream/render.py, optim.py:113-268)
  adam      batch-averaged Adam with fp64 moments (ref optim.py:281-407)
  dynamics  light visibility and rigid object transforms
            (ref render.py:350-368, model.py:539-572)
"""
