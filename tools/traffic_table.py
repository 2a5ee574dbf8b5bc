"""Build profiles/traffic.json from ncu launch captures of the persistent
streaming launch at each shard size (scripts/gpu_r2_f.sh: --metrics
dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum on the
fs_step_many launch of 20 steps).  bench.py reads the table for the line's
`roofline.traffic` and its L2 label (DRAM / algorithmic < 0.9 = L2-assisted).

    python tools/traffic_table.py gpurun_out/traffic > profiles/traffic.json
"""
import csv
import glob
import json
import os
import sys

BYTES = {"cfg1": 120, "cfg2": 120, "cfg3": 121, "cfg4": 160}
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
        m = {r[12]: float(r[14]) for r in rows}
        if "dram__bytes_read.sum" not in m:
            continue
        dram = (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / steps
        alg = BYTES[cfg] * int(n)
        out[key] = {"kernel": rows[0][4], "dram_bytes_per_step": dram,
                    "dram_read_per_step": m["dram__bytes_read.sum"] / steps,
                    "dram_write_per_step": m["dram__bytes_write.sum"] / steps,
                    "algorithmic_bytes_per_step": alg, "dram_over_algorithmic": dram / alg,
                    "ncu_us_per_step": m["gpu__time_duration.sum"] / steps / 1e3,
                    "source": f"profiles/raw/r2_traffic/{os.path.basename(path)} (ncu --metrics "
                              "dram bytes, --clock-control none, " +
                              (f"one fs_step_many launch of {STEPS} steps)" if steps > 1 else
                               "one fs_step launch of the K-launch graph)")}
    json.dump(out, sys.stdout, indent=1, sort_keys=True)
    print()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/traffic")
