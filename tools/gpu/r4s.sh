timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r4s_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r4s_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4s_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r4s_smoke.log
