# Per-kernel device durations (ncu launch list, one metric, clocks uncontrolled) for one bench step.
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && tail -n 1 gpurun_out/plain.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', round(d['ms_per_step'],3), 'fwd', round(d['roofline']['fwd']['ms'],3), 'bwd', round(d['roofline']['bwd_ms'],3))"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_bwd|attn_fwd|k_ffd|k_gather|k_scatter|k_token" --csv --log-file gpurun_out/klist.csv $CMD > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/klist.csv")) if len(r) > 10]
tot = 0.0
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ii = h.index("ID")
last = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki].replace("<unnamed>::", "").split("(")[0].replace("void ", "")
    last.setdefault(name, []).append(float(r[vi].replace(",", "")) / 1000)
for k, v in last.items():
    print(f"{k:40s} last={v[-1]:8.1f} us  (n={len(v)})")
PY
