# Final multi-GPU evidence at HEAD (W = all GPUs of the box): multi-rank parity, default bench line
set -x
N=$(nvidia-smi -L | wc -l)
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29721 tests/multi_rank_parity.py > gpurun_out/final_mg_parity_n$N.log 2>&1; echo parity rc $?
RALPB_TIMELINE_OUT=gpurun_out/final_timeline_n$N.json timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29722 bench.py --gpus $N > gpurun_out/final_mg_bench_n$N.log 2>&1; echo bench rc $?
tail -n 2 gpurun_out/final_mg_parity_n$N.log; grep -h '^{' gpurun_out/final_mg_bench_n$N.log | tail -1 | cut -c1-300
