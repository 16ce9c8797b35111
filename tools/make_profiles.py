"""Summarise a measurement pass (tools/gpu_full.sh output in gpurun_out/) into profiles/<round>/.

  python tools/make_profiles.py [--round r01]

Writes ncu_launches.csv (raw launch list), step_breakdown.txt (one bench step's kernels, serialised
ncu durations), ncu_full_summary.txt (key metrics of the --set full capture) and ncu_traffic.json
(DRAM bytes per attention kernel, read by bench.py for roofline.traffic).
"""
import argparse
import collections
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import summary  # noqa: E402


def short(name):
    return name.replace("<unnamed>::", "").split("(")[0].replace("void ", "").strip()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--src", default=os.path.join(ROOT, "gpurun_out"))
    a = ap.parse_args()
    out = os.path.join(ROOT, "profiles", a.round)
    os.makedirs(out, exist_ok=True)
    launches = os.path.join(a.src, "launches.csv")
    if os.path.exists(launches):
        shutil.copy(launches, os.path.join(out, "ncu_launches.csv"))
        rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
        h = rows[0]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        names = [short(r[ki]) for r in rows[1:]]
        vals = [float(r[vi].replace(",", "")) / 1000 for r in rows[1:]]
        # one step = the launches after the last "k_init" (the packer's first kernel) of the run
        starts = [i for i, n in enumerate(names) if n == "k_init"]
        s0 = starts[-2] if len(starts) > 1 else 0
        s1 = starts[-1] if len(starts) > 1 else len(names)
        step = list(zip(names[s0:s1], vals[s0:s1]))
        tot = sum(v for _, v in step)
        with open(os.path.join(out, "step_breakdown.txt"), "w") as f:
            for n, v in step:
                f.write(f"{n:45s} {v:9.1f} us  {100 * v / tot:5.1f}%\n")
            f.write(f"total {tot:.1f} us (ncu launch list, serialised, cold-cache; one bench step)\n")
        print(open(os.path.join(out, "step_breakdown.txt")).read())
    rep = os.path.join(a.src, "prof_full.ncu-rep")
    if os.path.exists(rep):
        res = summary(rep)
        with open(os.path.join(out, "ncu_full_summary.txt"), "w") as f:
            for d in res:
                f.write(f"== {d['kernel']}\n")
                for k, v in d.items():
                    if k != "kernel":
                        f.write(f"  {k:78s} {v}\n")
        traffic = collections.OrderedDict()
        for d in res:
            def num(k):
                v = d.get(k, "0").split()
                x = float(v[0].replace(",", ""))
                unit = v[1] if len(v) > 1 else ""
                return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1.0, "us": 1e-3}.get(unit, 1.0)
            traffic[short(d["kernel"])] = {"dram_read_bytes": num("dram__bytes_read.sum"),
                                           "dram_write_bytes": num("dram__bytes_write.sum"),
                                           "duration_ms": num("gpu__time_duration.sum")}
        json.dump({"source": f"profiles/{a.round}/ncu_full_summary.txt (ncu --set full --clock-control none, "
                             "one bench step, config 2)", "kernels": traffic},
                  open(os.path.join(out, "ncu_traffic.json"), "w"), indent=1)
        print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
