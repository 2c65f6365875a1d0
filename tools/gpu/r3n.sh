timeout 120 ./tools/nvls_probe 2 > gpurun_out/r3n_nvls.txt 2>&1
echo "rc=$?" >> gpurun_out/r3n_nvls.txt
