# A/B of the CQ micro-panel path of qr_reg.cu: parity tests in every mode, panel times, trace
mkdir -p gpurun_out
for m in ${MODES:-1 2 3 0}; do
RUTV_QR_CQ=$m timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_randutv.py -x -q -k "hqr or apply_q or randutv or factor" > gpurun_out/cq_pytest_$m.log 2>&1; echo "mode $m pytest=$?"; tail -3 gpurun_out/cq_pytest_$m.log
done
for m in 0 1; do
RUTV_QR_CQ=$m timeout 600 python tools/time_hqr.py 128,128 512,128 1000,128 2000,128 3000,128 4000,128 2000,64 6000,256 > gpurun_out/cq_time_$m.jsonl 2>&1; echo time$m=$?
grep -v Warn gpurun_out/cq_time_$m.jsonl | cut -c1-110
done
RUTV_QR_TRACE=1 timeout 300 python tools/probe_hqr.py 2000 128 > gpurun_out/cq_trace_2000.log 2>&1; echo $?
grep -n "qr_reg trace\|mp \|phase [0-9]" gpurun_out/cq_trace_2000.log | head -18
