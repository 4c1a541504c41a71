timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -1
timeout 300 python tools/gemm_bench.py "wave" > gpurun_out/sweep8.jsonl
for i in 1 2; do REPS=3 PROFILE=0 timeout 300 python tools/probe_perf.py 4000,128,2 10000,256,1 2>&1 | tail -2; done
REPS=1 PROFILE=1 timeout 300 python tools/probe_perf.py 4000,128,2 2>&1 | tail -1
python tools/time_hqr.py 4000,128 2000,128 50000,512 50000,8 12500,512 10000,256 > gpurun_out/hqr2.jsonl 2>&1
