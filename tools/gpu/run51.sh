# GPU session 51: a third TMA producer warp for MN-major operands (backward-filter GEMMs)
set -x
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_branchy_gpu.py -q -x > gpurun_out/t_51.log 2>&1; echo tests rc $?
for pr in 2 3; do
  for sh in 147,32,32 147,32,64 73,96,192 35,64,96; do RALPB_GEMM_PRODUCERS=$pr timeout 120 python tools/probe_conv.py --shape $sh --op wgrad --iters 10 | sed "s/^/p$pr /"; done
done
for i in 1 2; do
  for pr in 2 3; do
    for mdl in inception-v3 resnet-50 googlenet vgg16; do
      RALPB_GEMM_PRODUCERS=$pr timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/p$pr /"
    done
  done
done
tail -2 gpurun_out/t_51.log
