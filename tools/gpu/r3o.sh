for G in 148 592 1184; do echo "G=$G N=4"; timeout 120 ./tools/nvls_probe 4 $G 2>&1 | grep rank | head -2; done > gpurun_out/r3o_nvls.txt
echo "N=2" >> gpurun_out/r3o_nvls.txt; timeout 120 ./tools/nvls_probe 2 592 2>&1 | grep rank | head -1 >> gpurun_out/r3o_nvls.txt
