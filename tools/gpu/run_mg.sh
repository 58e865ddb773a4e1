# Multi-GPU session: the multi-rank parity script (W = all GPUs of the box) and the bench at N
set -x
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29631 tests/multi_rank_parity.py > gpurun_out/mg_parity_n$N.log 2>&1; echo parity rc $?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29632 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/mg_bench_n$N.log 2>&1; echo bench rc $?
tail -n 5 gpurun_out/mg_parity_n$N.log
grep -h '^{' gpurun_out/mg_bench_n$N.log | tail -c 3000
