set -x
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r2s_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2s_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err
OOCNMF_FUSED=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r2s_bench_twopass.json 2>> gpurun_out/r2s_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2s_launches.csv python bench.py --steps 2 --warmup 3 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r2s_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mu_fused -s 3 -c 1 -o gpurun_out/r2s_fused python bench.py --steps 2 --warmup 3 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r2s_ncu_full.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_smoke.log
