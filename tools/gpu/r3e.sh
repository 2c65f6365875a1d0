(for D in 1 2 3; do for K in 1/1 3/4 2/3 1/2 1/3 0/1; do for P in 0 1; do
echo "D=$D KEEP=$K POL=$P: $(OOCNMF_FUSED_KEEP=$K timeout 60 ./tools/fz_time 32 65536 65536 $D 10 $P | grep 'ms per' | sed 's/.*: //')"
done; done; done
) > gpurun_out/r3e_keep.txt 2>&1
