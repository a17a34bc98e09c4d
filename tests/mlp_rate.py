"""Debug: achieved TFLOP/s of each fused-MLP launch class in one forward of config CFG (default c5; CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_26580_b200 as P
cfg = P.configs()[os.environ.get("CFG", "c5")]
wl, m = cfg.workload, cfg.model
e = wl.code()
nb = int(os.environ.get("BINS", "512"))
_, S = wl.bins(e, 0, nb)
ctx = P.Context(m, P.weights_init(m, 1), e, wl.checks, wl.slots)
X = np.full((nb, wl.k, wl.slots), -1, np.int32)
ctx.denoise(X, S)
ctx.reset_stats()
ctx.set_profiling(True)
for _ in range(3):
    ctx.denoise(X, S)
st = ctx.kernel_stats()
tot = sum(v["ms"] for v in st.values())
for k, v in sorted(st.items(), key=lambda kv: -kv[1]["ms"]):
    tf = v["flops"] / (v["ms"] / 1e3) / 1e12 if v["ms"] else 0
    print(f"{k:16s} {v['ms']:8.3f} ms {100*v['ms']/tot:5.1f}%  {tf:7.1f} TF/s  launches {v['launches']}")
