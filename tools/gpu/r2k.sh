set -x
(for d in 1 2; do for p in 0 1 2; do timeout 60 ./tools/fz_time 32 65536 65536 $d 10 $p; done; done) > gpurun_out/r2k_fz.txt 2>&1
timeout 60 ./tools/tc_stall 32 65536 65536 1 5 > gpurun_out/r2k_tc_stall.txt 2>&1
for cfg in "2 0" "2 1" "1 1"; do set -- $cfg
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_mu_fused -c 1 ./tools/fz_time 32 65536 65536 $1 2 $2 > gpurun_out/r2k_ncu_d$1_p$2.log 2>&1
done
