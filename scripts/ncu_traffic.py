#!/usr/bin/env python
"""Average per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
and duration of each kernel in ncu reports covering one frame's launches.
Prints JSON keyed "<workload>_<stage>_fp16" as bench.py's roofline.traffic
expects (bench.py looks up f"{workload}_{dominant}_{precision}").

  python scripts/ncu_traffic.py [--workload c2] report.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys

STAGE = {"k_mlp_tc": "mlp", "k_march": "march", "k_place": "scatter"}


def main(argv):
    wl = "c2"
    if argv and argv[0] == "--workload":
        wl, argv = argv[1], argv[2:]
    paths = argv
    out = {"how": f"ncu --set full --clock-control none, every launch of one {wl.upper()} frame (bench.py --steps 1 "
                  "--warmup 1), mean over launches of dram__bytes_read.sum + dram__bytes_write.sum"}
    for p in paths:
        raw = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h = rows[0]
        data = [r for r in rows[2:] if len(r) == len(h)]
        name = next((v for k, v in STAGE.items() if k in data[0][h.index("Kernel Name")]), None) if data else None
        if not name:
            continue

        def col(m):
            i = h.index(m)
            unit = rows[1][i]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
                     "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(unit, 1)
            return [float(r[i].replace(",", "")) * scale for r in data]

        rd, wr, dur = col("dram__bytes_read.sum"), col("dram__bytes_write.sum"), col("gpu__time_duration.sum")
        n = len(data)
        out[f"{wl}_{name}_fp16"] = (sum(rd) + sum(wr)) / n
        out[f"{wl}_{name}_detail"] = {"launches": n, "dram_read_per_launch": sum(rd) / n,
                                      "dram_write_per_launch": sum(wr) / n, "mean_duration_us": 1e6 * sum(dur) / n}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
