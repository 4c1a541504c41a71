# bench line + torchrun paths + ncu launch list + ncu --set full GEMM sample for the committed profiles/
timeout 600 python bench.py > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; echo bench=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tr.json 2> gpurun_out/bench_tr.err; echo torchrun=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --sharded --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_trs.json 2> gpurun_out/bench_trs.err; echo torchrun_sharded=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_g.csv python tools/one_factorization.py 4000 128 2 > gpurun_out/launches_g.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none -k regex:dgemm_kernel --launch-skip 760 -c 40 -o gpurun_out/gemm_full_g python tools/one_factorization.py 4000 128 2 > gpurun_out/gemm_full_g.log 2>&1; echo ncu2=$?
