# GPU session 48: max-pool gather backward at a full SM of threads
set -x
timeout 1500 python -m pytest tests/test_kernels_gpu.py tests/test_branchy_gpu.py -q -x > gpurun_out/t_48.log 2>&1; echo tests rc $?
for i in 1 2; do
  for b in 4 8 16; do
    RALPB_POOL_GATHER_BLOCKS=$b timeout 300 python tools/model_launches.py inception-v3 6 2>/dev/null | sed "s/^/b$b /"
    RALPB_POOL_GATHER_BLOCKS=$b timeout 300 python tools/model_launches.py alexnet 6 2>/dev/null | sed "s/^/b$b /"
  done
done
timeout 300 python tools/gemm_probe.py inception-v3 12 > gpurun_out/gemm_probe_inc48.txt 2>&1
tail -2 gpurun_out/t_48.log
