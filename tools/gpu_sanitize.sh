# compute-sanitizer over tools/sanitize_cases.py (each tool bounded by its own timeout).
mkdir -p gpurun_out
timeout -s KILL 120 python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 7 python tools/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases ok|Error" gpurun_out/san_$tool.log | head -5
done
