set -x
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r3a_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3a_smoke.log 2>&1
PYTHONPATH=. timeout 600 python tools/fused_crossover.py --d=1,2 --k=16,32 16384x32768 32768x32768 > gpurun_out/r3a_cross.jsonl 2>&1
timeout 900 python bench.py --workload select --steps 20 --warmup 3 > gpurun_out/r3a_select.json 2> gpurun_out/r3a_select.err
timeout 900 python bench.py > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err
