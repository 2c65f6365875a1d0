set -x
timeout 1500 python -m pytest tests/test_multi_gpu.py tests/test_gpu_distributed.py -q -rf -p no:cacheprovider > gpurun_out/r3r_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3r_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r3r_bench_n4.json 2> gpurun_out/r3r_bench_n4.err
