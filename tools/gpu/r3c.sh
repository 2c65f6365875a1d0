set -x
nvidia-smi -L > gpurun_out/r3c_gpus.txt
timeout 900 python -m pytest tests/test_cli_gpu.py tests/test_gpu_distributed.py -q -rf -p no:cacheprovider > gpurun_out/r3c_cli2.log 2>&1
echo "rc=$?" >> gpurun_out/r3c_cli2.log
