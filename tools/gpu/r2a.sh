set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r2a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 300 ./tools/l2_probe > gpurun_out/r2a_l2probe.txt 2>&1
(timeout 120 ./tools/tc_stall 32 2048 8192 1 400; timeout 120 ./tools/tc_stall 32 4096 8192 1 200; timeout 120 ./tools/tc_stall 32 65536 65536 1 5) > gpurun_out/r2a_tcstall.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
echo "bench rc=$?" >> gpurun_out/r2a_bench.err
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2a_ref.json 2> gpurun_out/r2a_ref.err
echo "ref rc=$?" >> gpurun_out/r2a_ref.err
