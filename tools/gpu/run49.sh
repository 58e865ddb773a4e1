# GPU session 49: 16-aligned wide channels zero-extended onto the implicit path (Inception's 80-channel 3x3)
set -x
timeout 1500 python -m pytest tests/test_branchy_gpu.py -q -x > gpurun_out/t_49.log 2>&1; echo tests rc $?
for i in 1 2; do
  for c in 64 0; do
    RALPB_MODULE_CPAD_MIN=$c timeout 300 python tools/model_launches.py inception-v3 6 2>/dev/null | sed "s/^/cpad$c /"
    RALPB_MODULE_CPAD_MIN=$c timeout 300 python tools/model_launches.py googlenet 6 2>/dev/null | sed "s/^/cpad$c /"
  done
  RALPB_MODULE_CPAD_MIN=48 timeout 300 python tools/model_launches.py inception-v3 6 2>/dev/null | sed "s/^/cpad48 /"
  RALPB_MODULE_CPAD_MIN=200 timeout 300 python tools/model_launches.py googlenet 6 2>/dev/null | sed "s/^/cpad200 /"
done
timeout 300 python tools/gemm_probe.py inception-v3 12 > gpurun_out/gemm_probe_inc49.txt 2>&1
tail -2 gpurun_out/t_49.log
