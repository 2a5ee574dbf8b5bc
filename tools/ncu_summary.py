"""Per-step summary of an ncu `--page raw --csv` export of the hot kernel.

python tools/ncu_summary.py RAW.csv CONFIG VEHICLES STEPS ALG_BYTES_PER_VEHICLE_STEP [--merge]

STEPS is the number of control steps the captured launch streamed (the
persistent fs_step_many launch runs all K steps; 1 for a per-step fs_step
launch).  Prints a JSON object (and with --merge writes it into
profiles/ncu_summary.json under CONFIG, the file bench.py reads `traffic`
from): DRAM bytes per step, thread instructions per vehicle-step, issue /
DRAM utilisation, registers, grid and block.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = {
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "duration_ns": "gpu__time_duration.sum",
    "thread_inst": "thread_inst_executed",
    "issue_active": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1,
              "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9}


def read(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    i = rows.index(hdr)
    units, vals = rows[i + 1], rows[i + 2]
    out = {"kernel": vals[hdr.index("Kernel Name")]}
    for key, name in METRICS.items():
        if name not in hdr:
            continue
        j = hdr.index(name)
        v = float(vals[j].replace(",", ""))
        out[key] = v * UNIT_SCALE.get(units[j], 1)
    return out


def main():
    raw, config, n, steps, alg = sys.argv[1:6]
    n, steps, alg = int(n), int(steps), float(alg)
    m = read(raw)
    per_step = (m["dram_read"] + m["dram_write"]) / steps
    s = {
        "kernel": m["kernel"],
        "steps_in_launch": steps,
        "dram_read_bytes": m["dram_read"] / steps,
        "dram_write_bytes": m["dram_write"] / steps,
        "dram_bytes_per_launch": per_step,
        "algorithmic_bytes_per_launch": alg * n,
        "ncu_duration_us_per_step": m["duration_ns"] / steps / 1e3,
        "thread_inst_per_vehicle": m.get("thread_inst", 0) / steps / n,
        "issue_active_pct": m.get("issue_active"),
        "dram_throughput_pct": m.get("dram_pct"),
        "registers": m.get("registers"),
        "grid": m.get("grid"),
        "block": m.get("block"),
        "note": ("per control step: the captured launch streamed %d steps (fs_step_many); "
                 "'dram_bytes_per_launch' is per step, the unit bench.py's roofline uses" % steps
                 if steps > 1 else "one fs_step launch"),
        "source": os.path.relpath(raw, ROOT),
    }
    print(json.dumps(s, indent=1))
    if "--merge" in sys.argv:
        path = os.path.join(ROOT, "profiles", "ncu_summary.json")
        cur = json.load(open(path)) if os.path.exists(path) else {}
        cur[config] = s
        with open(path, "w") as f:
            json.dump(cur, f, indent=1)
            f.write("\n")


if __name__ == "__main__":
    main()
