# GPU session 47: unrolled k3/s2 max-pool backward gather; 16-aligned wide channels on the implicit path
set -x
timeout 1500 python -m pytest tests/test_branchy_gpu.py tests/test_kernels_gpu.py -q -x > gpurun_out/t_47.log 2>&1; echo tests rc $?
RALPB_MODULE_IMPLICIT_C16=64 timeout 1500 python -m pytest tests/test_branchy_gpu.py -q -x > gpurun_out/t_47b.log 2>&1; echo tests c16 rc $?
for i in 1 2; do
  timeout 300 python tools/model_launches.py inception-v3 6 2>/dev/null | sed "s/^/base /"
  RALPB_MODULE_IMPLICIT_C16=64 timeout 300 python tools/model_launches.py inception-v3 6 2>/dev/null | sed "s/^/c16_64 /"
  RALPB_MODULE_IMPLICIT_C16=16 timeout 300 python tools/model_launches.py inception-v3 6 2>/dev/null | sed "s/^/c16_16 /"
  timeout 300 python tools/model_launches.py googlenet 6 2>/dev/null | sed "s/^/base /"
  RALPB_MODULE_IMPLICIT_C16=64 timeout 300 python tools/model_launches.py googlenet 6 2>/dev/null | sed "s/^/c16_64 /"
  timeout 300 python tools/model_launches.py alexnet 6 2>/dev/null | sed "s/^/base /"
done
RALPB_MODULE_IMPLICIT_C16=64 timeout 300 python tools/gemm_probe.py inception-v3 30 > gpurun_out/gemm_probe_inc47.txt 2>&1
tail -2 gpurun_out/t_47.log gpurun_out/t_47b.log
