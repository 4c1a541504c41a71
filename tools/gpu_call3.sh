# QR / Jacobi ncu captures + CholQR A/B on config 2
set -x
python tools/time_hqr.py 2000,128 4000,128 > gpurun_out/hqr_hh.jsonl 2>&1
RUTV_CHOLQR=1 python tools/time_hqr.py 2000,128 4000,128 > gpurun_out/hqr_chol.jsonl 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_hh.json 2>/dev/null
RUTV_CHOLQR=1 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_chol.json 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hqr_reg_kernel -s 4 -c 2 -o gpurun_out/ncu_hqr python tools/one_factorization.py > gpurun_out/ncu_hqr.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi_kernel -c 1 -o gpurun_out/ncu_jacobi python tools/one_factorization.py > gpurun_out/ncu_jacobi.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:form_t -s 4 -c 1 -o gpurun_out/ncu_formt python tools/one_factorization.py > gpurun_out/ncu_formt.log 2>&1
ls -la gpurun_out
