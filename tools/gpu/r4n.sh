timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29781 bench.py --gpus 4 --workload select --steps 20 --warmup 3 > gpurun_out/r4n_select4.json 2> gpurun_out/r4n_select4.err
timeout 900 python bench.py --workload select --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r4n_select1.json 2> gpurun_out/r4n_select1.err
