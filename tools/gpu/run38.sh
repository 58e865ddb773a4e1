# GPU session 38: implicit-GEMM 3x3 / 5x5 'same' branch-group convolutions (padded copies + conv.cuh kernels)
set -x
timeout 1500 python -m pytest tests/test_branchy_gpu.py -q -x > gpurun_out/t_38.log 2>&1; echo tests rc $?
for i in 1 2; do for v in 1 0; do for mdl in inception-v3 googlenet; do
  RALPB_MODULE_IMPLICIT=$v timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/implicit=$v /"
done; done; done
tail -3 gpurun_out/t_38.log
