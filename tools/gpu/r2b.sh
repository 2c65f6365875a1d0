# fused-kernel bring-up: targeted tests first (short timeouts), then the full GPU suite and a bench
set -x
timeout 300 python -m pytest tests/test_gpu_parity_r2.py -k "fused" -x -q -p no:cacheprovider > gpurun_out/r2b_fused.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_fused.log
timeout 1200 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r2b_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-sparse > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
for d in 1 3; do OOCNMF_FUSED_D=$d timeout 300 python bench.py --steps 20 --warmup 5 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r2b_bench_d$d.json 2>> gpurun_out/r2b_bench.err; done
OOCNMF_FUSED=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r2b_bench_twopass.json 2>> gpurun_out/r2b_bench.err
