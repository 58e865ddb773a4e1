# GPU session 64: SIMD byte-compare max-pool gather backward
set -x
timeout 1500 python -m pytest tests/test_kernels_gpu.py tests/test_step_gpu.py tests/test_branchy_gpu.py -q -x > gpurun_out/t_64.log 2>&1; echo tests rc $?
for i in 1 2; do
  for mdl in inception-v3 alexnet; do
    timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/new /"
    RALPB_LIB=abtest/base_pg.so timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/base /"
  done
done
timeout 300 python tools/gemm_probe.py inception-v3 6 > gpurun_out/gemm_probe_inc64.txt 2>&1
tail -2 gpurun_out/t_64.log
