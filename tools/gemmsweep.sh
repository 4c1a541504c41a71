for c in 0 1 2 3; do echo "scfg $c"; RUTV_GEMM_SCFG=$c timeout 200 python tools/probe_gemm.py 2>&1 | grep -E '"N": 128|"M": 128'; done
RUTV_GEMM_SCFG=0 timeout 300 python tools/probe_perf.py 4000,128,2 2>&1 | tail -1
