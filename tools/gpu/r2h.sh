set -x
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r2h_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2h_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err
OOCNMF_FUSED=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r2h_bench_twopass.json 2>> gpurun_out/r2h_bench.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r2h_bench_fused2.json 2>> gpurun_out/r2h_bench.err
