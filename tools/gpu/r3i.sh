# 4 GPUs: sparse config-3 N=4 under NCCL channel / algorithm variants
set -x
run() {  # tag env...
  tag=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29800 + RANDOM % 100)) bench.py --gpus 4 --workload sparse --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3i_$tag.json 2> gpurun_out/r3i_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/r3i_$tag.json'));print('$tag', round(d['value'],1), {k:round(v,3) for k,v in d['roofline']['per_kernel_ms'].items()})" >> gpurun_out/r3i_summary.txt 2>&1
}
run base NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING
run ch8 NCCL_MAX_NCHANNELS=8
run ch16 NCCL_MAX_NCHANNELS=16
run rs1 OOCNMF_RS_CHUNKS=1
run rs8 OOCNMF_RS_CHUNKS=8
run nvls0 NCCL_NVLS_ENABLE=0
grep -i "nvls\|multicast" gpurun_out/r3i_base.err | head -20 > gpurun_out/r3i_nvls.txt
