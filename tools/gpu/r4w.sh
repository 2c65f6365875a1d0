set -x
timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r4w_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r4w_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4w_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r4w_smoke.log
timeout 900 python bench.py > gpurun_out/r4w_bench.json 2> gpurun_out/r4w_bench.err
