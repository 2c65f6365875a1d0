set -x
(for i in 1 2 3; do
echo "prev: $(timeout 60 ./tools/fz_time_prev 32 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"
echo "grouped: $(timeout 60 ./tools/fz_time 32 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"
done
echo "kp16 prev: $(timeout 60 ./tools/fz_time_prev 16 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"
echo "kp16 grouped: $(timeout 60 ./tools/fz_time 16 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"
timeout 60 ./tools/fz_stall 32 65536 65536 1 10 0
) > gpurun_out/r3w_group.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity_r2.py -q -rf -p no:cacheprovider -k "fused or config2 or eta" > gpurun_out/r3w_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3w_pytest.log
