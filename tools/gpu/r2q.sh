for i in 1 2; do
timeout 60 ./tools/fz_stall_prev 32 65536 65536 1 5 0 | grep -E "ms per launch|latency|W ready|wait count" | sed 's/^/spin /'
timeout 60 ./tools/fz_stall 32 65536 65536 1 5 0 | grep -E "ms per launch|latency|W ready|wait count" | sed 's/^/ilp  /'
done > gpurun_out/r2q_ab.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity_r2.py -k "fused" -q -p no:cacheprovider > gpurun_out/r2q_fused.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_fused.log
