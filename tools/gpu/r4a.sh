timeout 1500 python -m pytest tests/test_multi_gpu.py -q -rf -p no:cacheprovider > gpurun_out/r4a_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r4a_pytest.log
