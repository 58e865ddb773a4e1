# GPU session 65: a fourth TMA producer warp (warp 12) for MN-major operands
set -x
timeout 1200 python -m pytest tests/test_kernels_gpu.py -q -x > gpurun_out/t_65.log 2>&1; echo tests rc $?
RALPB_GEMM_PRODUCERS=4 timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_branchy_gpu.py -q -x > gpurun_out/t_65b.log 2>&1; echo tests4 rc $?
for pr in 3 4; do
  for sh in 147,32,32 147,32,64 73,96,192 35,64,96; do RALPB_GEMM_PRODUCERS=$pr timeout 120 python tools/probe_conv.py --shape $sh --op wgrad --iters 10 | grep h= | sed "s/^/p$pr /"; done
done
for i in 1 2; do
  for pr in 3 4; do
    for mdl in inception-v3 resnet-50 googlenet vgg16; do
      RALPB_GEMM_PRODUCERS=$pr timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/p$pr /"
    done
  done
done
tail -2 gpurun_out/t_65.log gpurun_out/t_65b.log
