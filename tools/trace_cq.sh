mkdir -p gpurun_out
tools/microbench/chain16_mb
RUTV_QR_CQ=${CQ:-1} timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "hqr" 2>&1 | tail -2
RUTV_QR_TRACE=1 timeout 300 python tools/probe_hqr.py 2000 128 > gpurun_out/cq_trace_2000.log 2>&1; echo $?
grep -n "qr_reg trace\|mp \|phase [0-9]" gpurun_out/cq_trace_2000.log | head -17
timeout 600 python tools/time_hqr.py 128,128 1000,128 2000,128 4000,128 6000,256 2>&1 | grep -v Warn | cut -c1-110
