"""Per-stage DRAM traffic per launch from an ncu --csv launch list.

    python tools/ncu_traffic.py gpurun_out/<launches>.csv > profiles/traffic.json

Maps each training-iteration stage to its kernels (summing kernels that make up
one stage) and averages dram__bytes_read.sum + dram__bytes_write.sum per launch.
bench.py reads profiles/traffic.json for the roofline "traffic" field.
"""
import collections
import csv
import json
import sys

STAGES = {
    "proj_forward": ["k_bspmm<4, 0,"],
    "proj_adjoint_tv": ["k_bspmm<4, 1,"],
    "loss_fused": ["k_ssim_stats11<1>", "k_loss_grad11"],
    "fvr_forward": ["k_fvr_fwd"],
    "fvr_backward": ["k_fvr_bwd"],
    "fvr_bin": ["k_bin_emit", "k_onesweep", "k_tile_starts"],
}

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        if d["Metric Name"] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d.get("Metric Unit", "byte"), 1)
        per[(d["ID"], d["Kernel Name"])]["bytes"] += v
    out = {}
    for stage, ks in STAGES.items():
        tot = 0.0
        for k in ks:
            vals = [x["bytes"] for (i, name), x in per.items() if k in name]
            if vals:
                tot += sum(vals) / len(vals)
        if tot:
            out[stage] = {"dram_bytes_per_launch": tot, "kernels": ks, "source": path.split("/")[-1]}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
