set -x
timeout 1500 python -m pytest tests/test_multi_gpu.py tests/test_gpu_distributed.py tests/test_cli_gpu.py -q -rf -p no:cacheprovider > gpurun_out/r4d_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r4d_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r4d_bench_n1.json 2> gpurun_out/r4d_bench_n1.err
for n in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2976$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r4d_bench_n$n.json 2> gpurun_out/r4d_bench_n$n.err
done
