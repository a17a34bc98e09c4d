"""Debug: per-chunk timeline of the fused MLP kernels, one forward of config CFG (default c3).

Needs the diagnostic build of the library:
  make -C paper_2605_26580_b200/csrc EXTRA=-DCIDER_MLP_TRACE OUT=../_lib_trace ../_lib_trace/libcider.so
  CIDER_LIB_DIR=$PWD/paper_2605_26580_b200/_lib_trace python tests/trace_mlp.py
"""
import os, sys
os.environ["CIDER_TRACE_MLP"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_26580_b200 as P
cfg = P.configs()[os.environ.get("CFG", "c3")]
wl, m = cfg.workload, cfg.model
m = P.Model(m=m.m, dim=m.dim, hidden=m.hidden, layers=1, heads=m.heads, precision=m.precision)
e = wl.code()
_, S = wl.bins(e, 0, 256)
ctx = P.Context(m, P.weights_init(m, 1), e, wl.checks, wl.slots)
X = np.full((256, wl.k, wl.slots), -1, np.int32)
ctx.denoise(X, S)
ctx.denoise(X, S)
