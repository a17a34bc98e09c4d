"""Create / use / destroy contexts in a loop and watch the device memory in use (nvidia-smi): a leak in
cider_destroy (workspace buffers, graphs, streams, tensor maps, NCCL) shows as a steady climb."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_26580_b200 as P


def used_mib():
    out = subprocess.run(["nvidia-smi", "--query-gpu=memory.used", "--format=csv,noheader,nounits", "-i", "0"],
                         capture_output=True, text=True).stdout
    return int(out.strip().splitlines()[0])


cfg = P.configs()["c2"]
wl, model = cfg.workload, cfg.model
e = wl.code()
w = P.weights_init(model, 1)
_, S = wl.bins(e, 0, 64)
sched = P.RevealSchedule(steps=3)
marks = {}
for i in range(121):
    ctx = P.Context(model, w, e, wl.checks, wl.slots)
    ctx.refine(S, wl.k, sched, P.RemaskConfig(rank_fraction=0.25))
    ctx.refine(S, wl.k, sched, P.RemaskConfig(rank_fraction=0.25))  # captured + replayed graph
    ctx.denoise(np.full((64, wl.k, wl.slots), -1, np.int32), S)
    dec = P.BpDecoder(wl.m, e, wl.checks, wl.slots)
    dec.close()
    ctx.close()
    if i in (20, 70, 120):
        marks[i] = used_mib()
        print(i, marks[i], "MiB", flush=True)
growth = marks[120] - marks[20]
print("growth over 100 create/destroy cycles:", growth, "MiB")
sys.exit(0 if growth <= 64 else 1)
