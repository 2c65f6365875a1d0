timeout 900 python -m pytest tests/test_cli_gpu.py -q -rf -p no:cacheprovider > gpurun_out/r4m_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r4m_pytest.log
