timeout 600 python -m pytest tests/test_gpu_parity_r2.py -k "wide" -q -rf -p no:cacheprovider > gpurun_out/r2u_wide.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_wide.log
timeout 300 python bench.py --k 128 --steps 10 --warmup 3 --no-sparse --no-e2e --no-cpu-baseline --m 16384 > gpurun_out/r2u_bench_k128.json 2> gpurun_out/r2u_bench_k128.err
