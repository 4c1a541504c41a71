# round-2 final evidence: config-2 launch list, ncu --set full of the panel-QR and Jacobi kernels
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_c2.csv python tools/one_factorization.py 4000 128 2 > gpurun_out/launches_c2.log 2>&1; echo ncu1=$?
python tools/ncu_summary.py launches gpurun_out/launches_c2.csv gpurun_out/launches_c2.json; echo sum1=$?
gzip -f gpurun_out/launches_c2.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hqr_reg --launch-skip 0 -c 1 -o gpurun_out/hqr_final python tools/probe_hqr.py 2000 128 > gpurun_out/ncu_hqr.log 2>&1; echo ncu2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi_blk --launch-skip 1 -c 1 -o gpurun_out/jac_final python tools/time_svd.py 128 > gpurun_out/ncu_jac.log 2>&1; echo ncu3=$?
ls -la gpurun_out/*.ncu-rep
python -c "
import json; d=json.load(open('gpurun_out/launches_c2.json')); print(d['total_kernel_ms'], d['launches']); [print(k) for k in d['kernels'][:9]]"
