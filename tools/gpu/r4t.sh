timeout 600 python -m pytest tests/test_gpu_parity_r2.py -q -rf -p no:cacheprovider -k "w_gram" > gpurun_out/r4t_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r4t_pytest.log
