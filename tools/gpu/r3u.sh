set -x
timeout 1500 python -m pytest tests/test_multi_gpu.py -q -rf -p no:cacheprovider -k "nvls" > gpurun_out/r3u_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3u_pytest.log
for i in 1 2; do
OOCNMF_NVLS=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2972$i bench.py --gpus 4 --steps 20 --warmup 5 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r3u_dense_nvls4_$i.json 2> gpurun_out/r3u_dense_nvls4_$i.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2973$i bench.py --gpus 4 --steps 20 --warmup 5 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r3u_dense_base4_$i.json 2> gpurun_out/r3u_dense_base4_$i.err
done
