timeout 600 python -m pytest tests/test_gpu_parity_r2.py -q -rf -p no:cacheprovider -k "paths" > gpurun_out/r4x_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r4x_pytest.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29791 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r4x_bench_n4.json 2> gpurun_out/r4x_bench_n4.err
