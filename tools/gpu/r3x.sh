set -x
for n in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2975$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r3x_bench_n$n.json 2> gpurun_out/r3x_bench_n$n.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29759 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > gpurun_out/r3x_ref_n4.json 2> gpurun_out/r3x_ref_n4.err
