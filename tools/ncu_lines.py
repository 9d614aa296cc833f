"""Per-CUDA-source-line warp-stall samples from an ncu report (captured with
--import-source on; the source file must exist at its build path when reading).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    hdr, rows = None, []
    for ln in csv.reader(io.StringIO(out)):
        if ln and ln[0] == "Line No":
            hdr = ln
            continue
        if hdr is None or not ln or not ln[0].isdigit():
            continue
        rows.append(ln)
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(f(r[si]) for r in rows) or 1.0
    rows.sort(key=lambda r: -f(r[si]))
    print(f"total samples {tot:.0f}")
    for r in rows[:top]:
        st = sorted(((f(r[i]), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
        sts = " ".join(f"{n}={100 * v / max(f(r[si]), 1):.0f}%" for v, n in st if v > 0)
        print(f"{100 * f(r[si]) / tot:5.1f}%  L{r[0]:>4s} inst={f(r[ie]) / 1e6:8.1f}M  {sts:40s} {r[1].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
