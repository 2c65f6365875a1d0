timeout 60 ./tools/fz_stall 32 65536 65536 1 10 0 > gpurun_out/r4i_stall.txt 2>&1
