# GPU session 28 (2 GPUs): per-rank launch timeline (overlap of the sync bucket / scatter / FC update)
set -x
N=$(nvidia-smi -L | wc -l)
RALPB_TIMELINE_OUT=gpurun_out/timeline_n$N.json timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29711 bench.py --gpus $N --steps 20 --warmup 5 --quick > gpurun_out/mg_bench28_n$N.log 2>&1; echo bench rc $?
grep -h '^{' gpurun_out/mg_bench28_n$N.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['overlap_rank0'], d['breakdown_ms_rank0'])"
