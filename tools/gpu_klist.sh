# Per-kernel device durations (ncu launch list, one metric, clocks uncontrolled) for one bench step.
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu ${BENCH_ARGS}"
$CMD > gpurun_out/plain.log 2>&1 && tail -n 1 gpurun_out/plain.log | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/klist.csv $CMD > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/klist.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
last = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki].replace("<unnamed>::", "").split("(")[0].replace("void ", "")
    last.setdefault(name, []).append(float(r[vi].replace(",", "")) / 1000)
for k, v in last.items():
    print(f"{k:45s} last={v[-1]:8.1f} us  (n={len(v)})")
PY
