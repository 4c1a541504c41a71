# full GPU suite + smoke + bench lines of configs 1-3 (config 5 is the default bench: tools/gpu_final.sh)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -14 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
for c in 1 2 3; do
timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo bench$c=$?
python - <<PY
import json
d = json.load(open("gpurun_out/bench_c$c.json"))
print({k: d[k] for k in ("value", "ms_per_step")}, d["e2e"]["ms_per_step"], d["roofline"]["step_frac_of_peak"], d["clocks"])
PY
done
