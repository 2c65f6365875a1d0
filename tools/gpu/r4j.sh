(for i in 1 2 3; do
echo "kp32 prev: $(timeout 60 ./tools/fz_time_prev 32 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"
echo "kp32 reuse: $(timeout 60 ./tools/fz_time 32 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"
echo "kp16 prev: $(timeout 60 ./tools/fz_time_prev 16 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"
echo "kp16 reuse: $(timeout 60 ./tools/fz_time 16 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"
done) > gpurun_out/r4j_reuse.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_parity.py -q -rf -p no:cacheprovider -k "fused or config2 or eta or config1 or k32 or k64 or ragged or tiny" > gpurun_out/r4j_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r4j_pytest.log
