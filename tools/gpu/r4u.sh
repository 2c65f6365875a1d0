timeout 600 python -m pytest tests/test_gpu_parity_r2.py -q -rf -p no:cacheprovider -k "deterministic" > gpurun_out/r4u_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r4u_pytest.log
