(for i in 1 2 3; do
echo "kp32 keep: $(timeout 60 ./tools/fz_time_prev 32 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"
echo "kp32 discard: $(timeout 60 ./tools/fz_time 32 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"
echo "kp16 keep: $(timeout 60 ./tools/fz_time_prev 16 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"
echo "kp16 discard: $(timeout 60 ./tools/fz_time 16 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"
done) > gpurun_out/r4c_discard.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r4c_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r4c_pytest.log
timeout 900 python bench.py > gpurun_out/r4c_bench.json 2> gpurun_out/r4c_bench.err
