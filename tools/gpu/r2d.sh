set -x
# fused kernel alone: timing (no profile) and per-role waits (profile build), D = 1..3, policies
for d in 1 2 3; do timeout 60 ./tools/fz_time 32 65536 65536 $d 10 0; done > gpurun_out/r2d_fz_time.txt 2>&1
for d in 1 2; do timeout 60 ./tools/fz_stall 32 65536 65536 $d 5 0; done > gpurun_out/r2d_fz_stall.txt 2>&1
timeout 60 ./tools/fz_time 32 65536 65536 2 10 1 >> gpurun_out/r2d_fz_time.txt 2>&1
timeout 60 ./tools/fz_time 32 65536 65536 1 10 2 >> gpurun_out/r2d_fz_time.txt 2>&1
# small: everything L2-resident (A 64 MB) -> SM-side rate
timeout 60 ./tools/fz_stall 32 2048 8192 2 100 0 >> gpurun_out/r2d_fz_stall.txt 2>&1
timeout 60 ./tools/fz_time 32 2048 8192 2 100 0 >> gpurun_out/r2d_fz_time.txt 2>&1
# ncu: one fused launch, full set (dram bytes, L2 hit rate, stalls)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mu_fused -c 1 -o gpurun_out/r2d_fused ./tools/fz_time 32 65536 65536 1 2 0 > gpurun_out/r2d_ncu.log 2>&1
