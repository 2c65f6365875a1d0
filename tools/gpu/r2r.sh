timeout 60 ./tools/fz_stall 32 65536 65536 1 5 0 > gpurun_out/r2r_fz.txt 2>&1
timeout 60 ./tools/fz_stall 32 65536 65536 1 5 0 >> gpurun_out/r2r_fz.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_parity.py -k "fused or config1 or k32 or config2 or long_k" -q -p no:cacheprovider > gpurun_out/r2r_fused.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_fused.log
