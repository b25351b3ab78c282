#!/bin/bash
# GPU encoder parity + timing against the host encoder.
python -m pytest tests/test_gpu_encoder.py -x -q 2>&1 | tail -15
DTANS_VERBOSE=1 python - <<'PY'
import time, numpy as np, paper_2603_01915_b200 as P
from paper_2603_01915_b200 import synth
for name, gen in [("laplacian g=2591 (2^25 nnz)", lambda: synth.laplacian_2d(2591)),
                  ("banded-32 2^22 rows (2^27 nnz)", lambda: synth.banded_rows(2**22, 0, 2**22, band=32)),
                  ("rmat scale 20 f32", lambda: synth.rmat(20, 16 << 20))]:
    m = gen()
    P.encode_matrix(m, device=0) if name.startswith("lap") else None
    t = time.time(); ch = P.encode_matrix(m); th = time.time() - t
    t = time.time(); cd = P.encode_matrix(m, device=0); td = time.time() - t
    print(f"{name}: nnz={m.nnz} host {th:.3f} s  device {td:.3f} s  identical={P.serialize(ch) == P.serialize(cd)}", flush=True)
PY
