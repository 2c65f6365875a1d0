set -x
timeout 1200 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_parity.py -q -rf -p no:cacheprovider > gpurun_out/r4v_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r4v_pytest.log
for i in 1 2; do for d in 1 0; do
OOCNMF_FUSED_HDEFER=$d timeout 600 python bench.py --steps 50 --warmup 5 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r4v_n1_d${d}_$i.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/r4v_n1_d${d}_$i.json'));print('N=1 hdefer=$d', round(d['value'],2), {k:round(v,4) for k,v in d['phase_ms_per_step'].items()})" >> gpurun_out/r4v_summary.txt
OOCNMF_FUSED_HDEFER=$d timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29800 + RANDOM % 90)) bench.py --gpus 4 --steps 50 --warmup 5 --no-sparse --no-e2e --no-cpu-baseline --no-weak > gpurun_out/r4v_n4_d${d}_$i.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/r4v_n4_d${d}_$i.json'));print('N=4 hdefer=$d', round(d['value'],2), {k:round(v,4) for k,v in d['phase_ms_per_step'].items()})" >> gpurun_out/r4v_summary.txt
done; done
