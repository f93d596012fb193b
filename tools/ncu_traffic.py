"""DRAM bytes per launch from the ncu reports of tools/ncu_traffic.sh.

    python tools/ncu_traffic.py gpurun_out/ncu_<name>.ncu-rep ...

Prints, per report, each profiled launch's kernel, duration and
dram__bytes_read.sum + dram__bytes_write.sum, and the per-step total (the
sum over the profiled launches, which is what bench.py's roofline.traffic
uses: its `achieved` is the dominant family's algorithmic work over the
family's summed launch time).  --write merges the totals into
profiles/traffic.json under <name>.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3, "ms": 1e-3}


def launches(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv",
                          "--metrics", ",".join(METRICS)], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, data = rows[0], rows[1], rows[2:]
    for r in data:
        rec = {"kernel": r[head.index("Kernel Name")][:60]}
        for m in METRICS:
            i = head.index(m)
            rec[m] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
        yield rec


def main():
    write = "--write" in sys.argv
    reps = [a for a in sys.argv[1:] if a != "--write"]
    path = os.path.join(ROOT, "profiles", "traffic.json")
    table = json.load(open(path)) if os.path.exists(path) else {}
    for rep in reps:
        name = os.path.basename(rep).removeprefix("ncu_").removesuffix(".ncu-rep")
        total = 0.0
        for rec in launches(rep):
            b = rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"]
            total += b
            print(f"{name}: {rec['kernel']:<60} {rec['gpu__time_duration.sum'] * 1e6:9.1f} us "
                  f"read {rec['dram__bytes_read.sum'] / 1e6:8.1f} MB "
                  f"write {rec['dram__bytes_write.sum'] / 1e6:8.1f} MB")
        print(f"{name}: total {total / 1e6:.1f} MB")
        table[name] = total
    if write:
        src = table.pop("source", "")
        table["source"] = src
        json.dump(table, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
