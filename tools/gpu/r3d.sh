(for i in 1 2; do
timeout 60 ./tools/fz_time 32 65536 65536 1 10 0 | grep "ms per"
OOCNMF_FUSED_PLAN=1 timeout 60 ./tools/fz_time 32 65536 65536 1 10 0 | grep "ms per"
done
OOCNMF_FUSED_PLAN=1 timeout 60 ./tools/fz_stall 32 65536 65536 1 10 0
timeout 60 ./tools/fz_time 16 65536 65536 1 10 0 | grep "ms per"
OOCNMF_FUSED_PLAN=1 timeout 60 ./tools/fz_time 16 65536 65536 1 10 0 | grep "ms per"
) > gpurun_out/r3d_plan.txt 2>&1
