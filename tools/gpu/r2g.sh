set -x
timeout 300 python -m pytest tests/test_gpu_parity_r2.py -k "fused" -x -q -p no:cacheprovider > gpurun_out/r2g_fused.log 2>&1
echo "rc=$?" >> gpurun_out/r2g_fused.log
for d in 1 2; do timeout 60 ./tools/fz_time 32 65536 65536 $d 10 0; done > gpurun_out/r2g_fz_time.txt 2>&1
for d in 1 2; do timeout 60 ./tools/fz_stall 32 65536 65536 $d 5 0; done > gpurun_out/r2g_fz_stall.txt 2>&1
