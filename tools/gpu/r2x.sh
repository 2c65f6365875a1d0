set -x
timeout 600 python -m pytest tests/test_multi_gpu.py -k "dead_rank" -q -rf -p no:cacheprovider > gpurun_out/r2x_dead.log 2>&1
echo "rc=$?" >> gpurun_out/r2x_dead.log
