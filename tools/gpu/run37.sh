# GPU session 37 (4 GPUs): stability -- 3000 timed steps of the N=4 headline step (flags / graphs / sync)
set -x
N=$(nvidia-smi -L | wc -l)
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29731 bench.py --gpus $N --steps 3000 --warmup 5 --quick > gpurun_out/stab_n$N.log 2>&1; echo bench rc $?
grep -h '^{' gpurun_out/stab_n$N.log | tail -1 | cut -c1-400
