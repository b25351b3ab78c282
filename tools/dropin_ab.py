"""Interleaved drop-in spmv timing for two libdtans builds (subprocesses)."""
import os, subprocess, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, time
sys.path.insert(0, %r)
import numpy as np
import paper_2603_01915_b200 as P
from paper_2603_01915_b200 import synth
m = synth.laplacian_2d(2591); c = P.encode_matrix(m); x, y = synth.vectors(m); c.device(0)
for _ in range(3): o = P.spmv(c, x, y)
ts = []
for _ in range(15):
    t0 = time.perf_counter(); o = P.spmv(c, x, y); ts.append((time.perf_counter() - t0) * 1e3)
ts.sort(); print("%%.3f" %% ts[len(ts) // 2])
''' % REPO
for rnd in range(3):
    for lab, lib in (("old", os.path.join(REPO, "variants/old/libdtans.so")), ("new", "")):
        env = dict(os.environ)
        if lib:
            env["DTANS_LIB"] = lib
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(lab, "drop-in median ms", r.stdout.strip() or r.stderr[-300:])
