(for i in 1 2 3 4; do
echo "keep: $(timeout 60 ./tools/fz_time_prev 32 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"
echo "discard: $(timeout 60 ./tools/fz_time 32 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"
done) > gpurun_out/r4b_discard.txt 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_mu_fused -c 2 ./tools/fz_time 32 65536 65536 1 1 0 > gpurun_out/r4b_ncu_discard.txt 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_mu_fused -c 2 ./tools/fz_time_prev 32 65536 65536 1 1 0 > gpurun_out/r4b_ncu_keep.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity_r2.py -q -rf -p no:cacheprovider -k "fused or config2 or eta" > gpurun_out/r4b_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r4b_pytest.log
