set -x
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r2y_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2y_pytest.log
timeout 900 python bench.py --workload select --steps 20 --warmup 3 > gpurun_out/r2y_select.json 2> gpurun_out/r2y_select.err
timeout 900 python bench.py --workload ooc --ooc-gb 24 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2y_ooc.json 2> gpurun_out/r2y_ooc.err
