set -x
timeout 300 python -m pytest tests/test_gpu_parity_r2.py -k "fused" -q -p no:cacheprovider > gpurun_out/r2c_fused.log 2>&1
echo "rc=$?" >> gpurun_out/r2c_fused.log
timeout 1200 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r2c_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2c_pytest.log
OOCNMF_PROFILE_IO=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-sparse > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
for d in 1 3; do OOCNMF_FUSED_D=$d timeout 300 python bench.py --steps 20 --warmup 5 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r2c_bench_d$d.json 2>> gpurun_out/r2c_bench.err; done
for p in 1 2; do OOCNMF_FUSED_POL=$p timeout 300 python bench.py --steps 20 --warmup 5 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r2c_bench_pol$p.json 2>> gpurun_out/r2c_bench.err; done
OOCNMF_FUSED=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r2c_bench_twopass.json 2>> gpurun_out/r2c_bench.err
