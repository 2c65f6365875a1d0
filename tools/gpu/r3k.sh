set -x
timeout 900 python -m pytest tests/test_gpu_selection.py tests/test_cli_gpu.py -q -rf -p no:cacheprovider -k "select" > gpurun_out/r3k_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3k_pytest.log
timeout 900 python bench.py --workload select --steps 20 --warmup 3 > gpurun_out/r3k_select.json 2> gpurun_out/r3k_select.err
