"""Per-source-line instruction / stall breakdown of an ncu report.

python tools/ncu_lines.py REPORT.ncu-rep|SOURCE.csv [units] [top]
(units: vehicles/rays the launch processed, for per-unit instruction counts)
"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    if rep.endswith(".csv"):      # an exported source page (--page source --csv)
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                              "cuda,sass"], capture_output=True, text=True).stdout
    cur, hdr, rows = None, None, []
    for r in csv.reader(txt.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        try:
            ti = float(r[hdr.index("Thread Instructions Executed")] or 0)
            st = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        rows.append((ti, st, cur, r[0], r[1].strip()))
    tot_i = sum(x[0] for x in rows) or 1
    tot_s = sum(x[1] for x in rows) or 1
    print(f"thread instructions {tot_i:.4e} ({tot_i / units:.1f} per unit), stall samples {tot_s:.0f}")
    byfile = {}
    for ti, st, f, *_ in rows:
        a = byfile.setdefault(f, [0, 0])
        a[0] += ti
        a[1] += st
    for f, (ti, st) in sorted(byfile.items(), key=lambda kv: -kv[1][0]):
        print(f"  {f:20s} {100 * ti / tot_i:5.1f}% instr {100 * st / tot_s:5.1f}% stalls "
              f"{ti / units:7.1f}/unit")
    rows.sort(reverse=True)
    for ti, st, f, ln, src in rows[:top]:
        print(f"{100 * ti / tot_i:5.1f}% {100 * st / tot_s:5.1f}% {ti / units:6.1f} {f}:{ln} {src[:80]}")


if __name__ == "__main__":
    main()
