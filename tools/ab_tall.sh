# A/B: tall-panel Cholesky-QR2 (default) vs Householder kernels only (RUTV_CHOLQR_MIN_ROWS=0)
mkdir -p gpurun_out
RUTV_CHOLQR_MIN_ROWS=0 timeout 600 python tools/ab_tall.py run hh > gpurun_out/ab_tall_hh.jsonl 2>&1; echo hh=$?
timeout 600 python tools/ab_tall.py run cq > gpurun_out/ab_tall_cq.jsonl 2>&1; echo cq=$?
timeout 600 python tools/ab_tall.py compare hh cq > gpurun_out/ab_tall_cmp.jsonl 2>&1; echo cmp=$?
cat gpurun_out/ab_tall_hh.jsonl gpurun_out/ab_tall_cq.jsonl gpurun_out/ab_tall_cmp.jsonl
for c in "5 4" "4 14" "3 39"; do set -- $c
RUTV_CHOLQR_MIN_ROWS=0 timeout 900 python tools/probe_phases.py $1 $2 > gpurun_out/phases_c$1_hh.json 2>&1; echo $?
timeout 900 python tools/probe_phases.py $1 $2 > gpurun_out/phases_c$1_cq.json 2>&1; echo $?
cat gpurun_out/phases_c$1_hh.json gpurun_out/phases_c$1_cq.json
done
