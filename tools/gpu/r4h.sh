(for i in 1 2; do for P in 0 1 2; do
echo "pol $P: $(timeout 60 ./tools/fz_time 32 65536 65536 1 10 $P | grep 'ms per' | sed 's/.*: //')"
done; done
for K in 7/8 3/4; do echo "keep $K: $(OOCNMF_FUSED_KEEP=$K timeout 60 ./tools/fz_time 32 65536 65536 1 10 0 | grep 'ms per' | sed 's/.*: //')"; done
) > gpurun_out/r4h_pol.txt 2>&1
