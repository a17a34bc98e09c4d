"""Write profiles/ncu_summary.json: DRAM bytes per unit of algorithmic work for the fused MLP kernels,
from one `ncu --set full` capture of tests/mlp_rate.py (c5 shapes, 512 bins, layer-2 gate/agg/fuse).

  python tools/make_ncu_summary.py <mlp.ncu-rep> <bins>

bench.py multiplies these by its own per-launch algorithmic FLOPs to fill roofline.traffic.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import rep  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_26580_b200 as P  # noqa: E402

path, bins = sys.argv[1], int(sys.argv[2])
cfg = P.configs()["c5"]
wl, m = cfg.workload, cfg.model
K, L, E, D, H = wl.k, wl.slots, wl.slots * wl.col_weight, m.dim, m.hidden
Ms, Me = bins * L * K, bins * E * K
flops = {"<512, 256, 2,": ("mlp_gate", 2.0 * Ms * H * (2 * D + D)),
         "<256, 256, 0,": ("mlp_agg", 2.0 * Me * H * (D + D)),
         "<512, 256, 3,": ("mlp_fuse", 2.0 * Ms * H * (2 * D + D))}
out = {"source": f"{os.path.basename(path)}: ncu --set full, tests/mlp_rate.py c5 {bins} bins", "kernels": {}}
for r in rep(path):
    for tag, (name, fl) in flops.items():
        if tag in r["kernel"]:
            dram = (float(r["dram_rd_MB"]) + float(r["dram_wr_MB"])) * 1e6  # ncu reports MB (1e6)
            out["kernels"][name] = {"dram_bytes": dram, "algorithmic_flops": fl, "dram_bytes_per_algo_unit": dram / fl,
                                    "time_us_under_ncu": float(r["time_us"]),
                                    "tcgen05_bf16_pct": float(r.get("tcgen05_bf16_pct", "nan")),
                                    "source": out["source"]}
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_summary.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
