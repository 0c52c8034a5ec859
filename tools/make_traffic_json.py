"""profiles/traffic.json from one `ncu --set full` capture per workload.

    python tools/make_traffic_json.py gpurun_out/p2d/ncu profiles/r02/ncu

Reads every ncu_<workload>_raw.csv (ncu -i rep --page raw --csv) in the given
directory: dram__bytes_read.sum + dram__bytes_write.sum of the captured
kernel launch, with the kernel name and the bench's algorithmic bytes for
the launch (bench.algorithmic_bytes; the capture runs the full workload, or
a step-shortened run for long ones -- DRAM traffic of the stepper does not
depend on the step count, the samples do).  bench.py copies `dram_bytes`
into roofline.traffic for the matching workload.
"""

import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}  # time -> ms


def read_raw(path):
    with open(path) as f:
        rows = list(csv.reader(io.StringIO(f.read())))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for h, u, v in zip(hdr, units, vals):
        try:
            out[h] = float(v.replace(",", "")) * UNITS.get(u, 1)
        except ValueError:
            out[h] = v
    return out


def main():
    src, dst = sys.argv[1], sys.argv[2]
    path = os.path.join(ROOT, "profiles", "traffic.json")
    with open(path) as f:
        table = json.load(f)
    for name in sorted(os.listdir(src)):
        if not (name.startswith("ncu_") and name.endswith("_raw.csv")):
            continue
        wl = name[len("ncu_"):-len("_raw.csv")]
        if wl not in bench.WORKLOADS:
            continue
        d = read_raw(os.path.join(src, name))
        rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
        if not isinstance(rd, float) or not isinstance(wr, float):
            continue
        w = bench.WORKLOADS[wl]
        table[wl] = {
            "kernel": d.get("Kernel Name"),
            "dram_read_bytes": int(rd), "dram_write_bytes": int(wr), "dram_bytes": int(rd + wr),
            "algorithmic_bytes": int(bench.algorithmic_bytes(w, w["orbits"])),
            "duration_ms": d.get("gpu__time_duration.sum")
            if isinstance(d.get("gpu__time_duration.sum"), float) else None,
            "source": "%s/ncu_%s_summary.txt (ncu --set full, one launch of the full workload)"
                      % (dst, wl),
        }
    with open(path, "w") as f:
        json.dump(table, f, indent=2)
        f.write("\n")
    print("\n".join(sorted(k for k in table if not k.startswith("_"))))


if __name__ == "__main__":
    main()
