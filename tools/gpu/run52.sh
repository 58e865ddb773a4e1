# GPU session 52: lane-parallel TMA issue of MN-major atoms
set -x
RALPB_GEMM_LANES=1 timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_branchy_gpu.py -q -x > gpurun_out/t_52.log 2>&1; echo tests rc $?
for ln in 0 1; do
  for sh in 147,32,32 147,32,64 73,96,192 35,64,96; do RALPB_GEMM_LANES=$ln timeout 120 python tools/probe_conv.py --shape $sh --op wgrad --iters 10 | grep h= | sed "s/^/l$ln /"; done
done
for i in 1 2; do
  for ln in 0 1; do
    for mdl in inception-v3 resnet-50 googlenet vgg16; do
      RALPB_GEMM_LANES=$ln timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/l$ln /"
    done
  done
done
tail -2 gpurun_out/t_52.log
