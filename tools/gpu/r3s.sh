set -x
timeout 1500 python -m pytest tests/test_multi_gpu.py tests/test_gpu_distributed.py -q -rf -p no:cacheprovider > gpurun_out/r3s_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3s_pytest.log
run() { tag=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29710 + RANDOM % 80)) bench.py --gpus 4 --workload sparse --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3s_$tag.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r3s_$tag.json'));print('$tag', round(d['value'],1), {k:round(v,3) for k,v in d['phase_ms_per_step'].items()})" >> gpurun_out/r3s_summary.txt; }
run u2c1 OOCNMF_NVLS_U=2
run u4c1 OOCNMF_NVLS_U=4
run u2c2 OOCNMF_NVLS_CTAS=2
run u4c2 OOCNMF_NVLS_U=4 OOCNMF_NVLS_CTAS=2
run u2c1b OOCNMF_NVLS_U=2
