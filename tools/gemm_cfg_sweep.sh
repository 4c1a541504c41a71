for i in 1 2; do REPS=3 PROFILE=0 timeout 300 python tools/probe_perf.py 4000,128,2 10000,256,1 2>&1 | tail -2; done
for i in 1 2; do RUTV_GEMM_PLAN=1 REPS=3 PROFILE=0 timeout 300 python tools/probe_perf.py 4000,128,2 2>&1 | tail -1; done
