# full GPU suite + smoke + default bench line + phase profiles (configs 1-3)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 python tools/probe_perf.py 2000,128,0 4000,128,2 10000,256,1 > gpurun_out/perf.jsonl 2>&1; echo perf=$?
