"""Write profiles/compress_dram_bytes.json (bench.py's roofline.traffic) from an
`ncu --set full` capture of one fwht2p launch, tagged with the sha of the kernel
source it was captured from (bench.py ignores it once the source changes).

    python tools/ncu_traffic.py gpurun_out/fwht2p_full.ncu-rep
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        if "fwht2p" not in name:
            continue

        def val(key):
            i = hdr.index(key)
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(units[i], 1)
            return float(vals[i].replace(",", "")) * scale

        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        dur = float(vals[hdr.index("gpu__time_duration.sum")].replace(",", ""))
        rec = {"kernel": name, "report": Path(path).name, "dram_bytes_read": rd, "dram_bytes_write": wr,
               "dram_bytes_per_launch": rd + wr, "ncu_duration": f"{dur} {units[hdr.index('gpu__time_duration.sum')]}",
               "kernel_source_sha": bench._kernel_source_sha()}
        bench.TRAFFIC_FILE.write_text(json.dumps(rec, indent=1) + "\n")
        print(json.dumps(rec))
        return
    raise SystemExit("no fwht2p launch in " + path)


if __name__ == "__main__":
    main(sys.argv[1])
