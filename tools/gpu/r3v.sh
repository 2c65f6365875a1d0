set -x
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r3v_pytest2.log 2>&1
echo "rc=$?" >> gpurun_out/r3v_pytest2.log
