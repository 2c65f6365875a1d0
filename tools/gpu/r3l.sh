for i in 1 2 3; do
OOCNMF_SELECT_OVERLAP=0 timeout 900 python bench.py --workload select --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r3l_serial$i.json 2>/dev/null
timeout 900 python bench.py --workload select --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r3l_overlap$i.json 2>/dev/null
done
