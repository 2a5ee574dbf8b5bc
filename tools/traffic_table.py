"""Build profiles/traffic.json from ncu launch captures of the persistent
streaming launch at each shard size (scripts/gpu_r2_f.sh: --metrics
dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum on the
fs_step_many launch of 20 steps).  bench.py reads the table for the line's
`roofline.traffic` and its L2 label (DRAM / algorithmic < 0.9 = L2-assisted).

    python tools/traffic_table.py gpurun_out/traffic > profiles/traffic.json

`<config>@<n>_steps.csv` files are per-step launch captures (World.step
configs: every launch of ONE step, summed -- the forest step is three
kernels); their key is `<config>@<n>/steps`.
"""
import csv
import glob
import json
import os
import sys

BYTES = {"cfg1": 120, "cfg2": 120, "cfg3": 121, "cfg4": 160, "world": 211, "vecenv": 211,
         "forest": None}     # forest: the line counts its own (tested / reset fractions)
STEPS = 20


def main(src):
    out = {}
    for path in sorted(glob.glob(os.path.join(src, "*.csv"))):
        key = os.path.basename(path)[:-4]
        steps = 1 if key.endswith("_steps") else STEPS      # per-step launch captures
        if key.endswith("_steps"):
            key = key[:-len("_steps")] + "/steps"
        cfg, n = key.split("/")[0].split("@")
        rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
        m, t = {}, {}
        for r in rows:          # summed over the capture's launches
            m[r[12]] = m.get(r[12], 0.0) + float(r[14])
            if r[12] == "gpu__time_duration.sum":
                t[r[4]] = t.get(r[4], 0.0) + float(r[14])
        if "dram__bytes_read.sum" not in m:
            continue
        dram = (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / steps
        alg = BYTES[cfg] * int(n) if BYTES[cfg] else None
        out[key] = {"kernel": max(t, key=t.get), "dram_bytes_per_step": dram,
                    "dram_read_per_step": m["dram__bytes_read.sum"] / steps,
                    "dram_write_per_step": m["dram__bytes_write.sum"] / steps,
                    "algorithmic_bytes_per_step": alg,
                    "dram_over_algorithmic": dram / alg if alg else None,
                    "ncu_us_per_step": m["gpu__time_duration.sum"] / steps / 1e3,
                    "source": f"profiles/raw/r2_traffic/{os.path.basename(path)} (ncu --metrics "
                              "dram bytes, --clock-control none, " +
                              (f"one fs_step_many launch of {STEPS} steps)" if steps > 1 else
                               f"the {len(rows) // 3} launch(es) of one step)")}
        if len(t) > 1:
            out[key]["kernels_us"] = {k[:60]: v / 1e3 for k, v in t.items()}
    json.dump(out, sys.stdout, indent=1, sort_keys=True)
    print()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/traffic")
