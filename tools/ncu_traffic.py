"""Per-rotation DRAM traffic of each kernel of one sweep batch from an ncu --set full report
(dram__bytes_read.sum + dram__bytes_write.sum), for bench.py's roofline `traffic` field.

    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep ROTATIONS_PER_LAUNCH > profiles/r2/ncu_traffic.json
"""
import csv
import io
import json
import subprocess
import sys


def main(rep, rot):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    ki = hdr.index("Kernel Name")
    ri, wi, ti = (hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum"),
                  hdr.index("gpu__time_duration.sum"))
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tscale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
    per, dur = {}, {}
    for r in rows[2:]:
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").strip()
        b = float(r[ri].replace(",", "")) * scale[units[ri]] + float(r[wi].replace(",", "")) * scale[units[wi]]
        per[name] = per.get(name, 0.0) + b / rot
        dur[name] = dur.get(name, 0.0) + float(r[ti].replace(",", "")) * tscale[units[ti]]
    print(json.dumps({"dram_bytes_per_rotation": per, "duration_ms_per_launch": dur, "source": rep,
                      "rotations_per_launch": rot}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
