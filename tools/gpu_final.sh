# Round evidence with the current code: GPU suite, smoke, bench line (config 2) + configs 1/3 lines,
# torchrun replica + sharded lines, ncu launch list of one factorization, ncu --set full of 40 GEMM launches.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err; echo bench=$?
timeout 600 python bench.py --config 1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench1=$?
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench3=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tr.json 2> gpurun_out/bench_tr.err; echo torchrun=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --sharded --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_trs.json 2> gpurun_out/bench_trs.err; echo torchrun_sharded=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_h.csv python tools/one_factorization.py 4000 128 2 > gpurun_out/launches_h.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none -k regex:dgemm_kernel --launch-skip 760 -c 40 -o /tmp/gemm_full_h python tools/one_factorization.py 4000 128 2 > gpurun_out/gemm_full_h.log 2>&1; echo ncu2=$?
# summaries on the box (the reports themselves exceed gpurun's 64 MiB return limit)
python tools/ncu_summary.py launches gpurun_out/launches_h.csv gpurun_out/launches_h.json; echo sum1=$?
python tools/ncu_summary.py full /tmp/gemm_full_h.ncu-rep gpurun_out/gemm_full_h.json; echo sum2=$?
gzip -f gpurun_out/launches_h.csv
ls -la gpurun_out
