set -x
(for i in 1 2; do
 timeout 60 ./tools/fz_time 32 65536 65536 1 10 0 2 0
 timeout 60 ./tools/fz_time 32 65536 65536 2 10 0 2 1
 timeout 60 ./tools/fz_time 32 65536 65536 1 10 0 2 1
 timeout 60 ./tools/fz_time 32 65536 65536 2 10 1 2 1
done) > gpurun_out/r2p_fz.txt 2>&1
timeout 60 ./tools/fz_stall 32 65536 65536 2 5 0 2 1 > gpurun_out/r2p_fz_stall.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_mu_fused -c 1 ./tools/fz_time 32 65536 65536 2 2 0 2 1 > gpurun_out/r2p_ncu.log 2>&1
OOCNMF_FUSED_P2FIRST=1 OOCNMF_FUSED_D=2 timeout 300 python -m pytest tests/test_gpu_parity_r2.py -k "fused or config2" -q -p no:cacheprovider > gpurun_out/r2p_fused.log 2>&1
echo "rc=$?" >> gpurun_out/r2p_fused.log
