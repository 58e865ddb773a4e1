# GPU session 53: third producer for K-major GEMMs; deeper rings for small stages
set -x
RALPB_GEMM_PRODUCERS_K=3 RALPB_GEMM_MAX_STAGES=12 timeout 1200 python -m pytest tests/test_kernels_gpu.py -q -x > gpurun_out/t_53.log 2>&1; echo tests rc $?
for i in 1 2; do
  for cfg in "2 8" "3 8" "2 12" "3 12"; do
    set -- $cfg
    for mdl in inception-v3 resnet-50 googlenet vgg16; do
      RALPB_GEMM_PRODUCERS_K=$1 RALPB_GEMM_MAX_STAGES=$2 timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/k$1s$2 /"
    done
  done
done
tail -2 gpurun_out/t_53.log
