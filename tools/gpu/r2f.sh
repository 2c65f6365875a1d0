set -x
for d in 1 2; do timeout 60 ./tools/fz_time 32 65536 65536 $d 10 0; done > gpurun_out/r2f_fz_time.txt 2>&1
for d in 1 2; do timeout 60 ./tools/fz_stall 32 65536 65536 $d 5 0; done > gpurun_out/r2f_fz_stall.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity_r2.py -k "fused or config2 or long_k" -q -p no:cacheprovider > gpurun_out/r2f_fused.log 2>&1
echo "rc=$?" >> gpurun_out/r2f_fused.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mu_fused -c 1 -o gpurun_out/r2f_fused ./tools/fz_time 32 65536 65536 1 2 0 > gpurun_out/r2f_ncu.log 2>&1
