mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_qr_cq.py tests/test_gpu_tallqr.py tests/test_gpu_grid.py tests/test_gpu_step_api.py -x -q > gpurun_out/pytest_new.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_new.log
for c in 2 3; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2953$c bench.py --gpus 1 --sharded --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_sharded_c$c.json 2> gpurun_out/bench_sharded_c$c.err; echo sharded$c=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_sharded_c$c.json')); print('sharded 1x1 config $c', d['ms_per_step'], d['config'].get('parallelism'))"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2.csv python tools/one_factorization.py 4000 128 2 > gpurun_out/launches_c2.log 2>&1; echo ncu1=$?
python tools/ncu_summary.py launches gpurun_out/launches_c2.csv gpurun_out/launches_c2.json; echo sum1=$?
gzip -f gpurun_out/launches_c2.csv
python -c "
import json; d=json.load(open('gpurun_out/launches_c2.json')); print(d['total_kernel_ms']); [print(k) for k in d['kernels'][:8]]"
