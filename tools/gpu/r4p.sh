set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r4p_launches.csv python bench.py --steps 2 --warmup 3 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r4p_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mu_fused -s 2 -c 1 -o gpurun_out/r4p_fused python bench.py --steps 2 --warmup 3 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r4p_ncu_full.log 2>&1
