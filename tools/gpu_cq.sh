mkdir -p gpurun_out
python tools/time_hqr.py 500,128 1000,128 2000,128 4000,128 > gpurun_out/hqr_hh.jsonl 2>&1
RUTV_CHOLQR=1 RUTV_DEBUG=1 python tools/time_hqr.py 500,128 1000,128 2000,128 4000,128 > gpurun_out/hqr_chol.jsonl 2>&1
RUTV_CHOLQR=1 RUTV_DEBUG=1 PROFILE=1 timeout 300 python tools/probe_perf.py 2000,128,0 4000,128,2 > gpurun_out/perf_chol.jsonl 2>gpurun_out/perf_chol.err
grep -c fallback gpurun_out/perf_chol.err
