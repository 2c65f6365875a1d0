set -x
timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r3t_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3t_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3t_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r3t_smoke.log
timeout 900 python bench.py > gpurun_out/r3t_bench.json 2> gpurun_out/r3t_bench.err
timeout 1500 python bench.py --impl reference > gpurun_out/r3t_ref.json 2> gpurun_out/r3t_ref.err
