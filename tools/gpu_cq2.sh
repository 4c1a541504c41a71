mkdir -p gpurun_out
timeout 300 python tools/debug_cholqr.py > gpurun_out/dbg_cq.log 2>&1; echo dbg=$?
RUTV_CHOLQR=1 timeout 300 python tools/time_hqr.py 500,128 1000,128 2000,128 4000,128 > gpurun_out/hqr_chol.jsonl 2>&1; echo th=$?
timeout 900 python -m pytest tests/test_gpu_cholqr.py tests/test_gpu_randutv.py tests/test_gpu_configs.py -x -q > gpurun_out/pt.log 2>&1; echo pt=$?
tail -30 gpurun_out/pt.log
RUTV_DEBUG=1 timeout 300 python tools/probe_perf.py 2000,128,0 4000,128,2 10000,256,1 > gpurun_out/perf_cq.jsonl 2>gpurun_out/perf_cq.err; echo perf=$?
