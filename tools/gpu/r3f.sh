(OOCNMF_FUSED_KEEP=1/2 timeout 60 ./tools/fz_stall 32 65536 65536 2 10 0 | head -16
OOCNMF_FUSED_KEEP=1/3 timeout 60 ./tools/fz_stall 32 65536 65536 3 10 0 | head -16
timeout 60 ./tools/fz_stall 32 65536 65536 1 10 0 | head -16
) > gpurun_out/r3f_stall.txt 2>&1
