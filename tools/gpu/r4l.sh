timeout 1500 python -m pytest tests/test_multi_gpu.py tests/test_gpu_distributed.py -q -rf -p no:cacheprovider > gpurun_out/r4l_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r4l_pytest.log
