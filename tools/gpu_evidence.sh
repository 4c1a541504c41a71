# bench line + ncu launch list + ncu --set full GEMM sample for the committed profiles/
timeout 600 python bench.py > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_e.csv python tools/one_factorization.py 4000 128 2 > gpurun_out/launches_e.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:dgemm_kernel --launch-skip 760 -c 40 -o gpurun_out/gemm_full_e python tools/one_factorization.py 4000 128 2 > gpurun_out/gemm_full_e.log 2>&1
ls -la gpurun_out | tail -5
