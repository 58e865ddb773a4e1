# GPU session 24 (2 GPUs): nvidia-smi NVLink counter probe + multi-rank parity regression
set -x
nvidia-smi nvlink -h > gpurun_out/nvl_help.txt 2>&1
nvidia-smi nvlink -gt d -i 0 > gpurun_out/nvl_gt0.txt 2>&1; echo gt rc $?
nvidia-smi nvlink -s -i 0 > gpurun_out/nvl_s0.txt 2>&1
nvidia-smi nvlink -e -i 0 > gpurun_out/nvl_e0.txt 2>&1; echo e rc $?
N=$(nvidia-smi -L | wc -l)
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29681 tests/multi_rank_parity.py > gpurun_out/mg_parity24_n$N.log 2>&1; echo parity rc $?
nvidia-smi nvlink -gt d -i 0 > gpurun_out/nvl_gt0_after.txt 2>&1
tail -n 2 gpurun_out/mg_parity24_n$N.log; head -30 gpurun_out/nvl_gt0.txt
