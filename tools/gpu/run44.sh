# GPU session 44: sibling 1x1 groups (one GEMM / stats pass / wgrad / dgrad per group),
# unrolled 3x3 avg pool windows, k3/s2 max-pool backward
set -x
timeout 1500 python -m pytest tests/test_branchy_gpu.py tests/test_resnet_gpu.py -q -x > gpurun_out/t_44.log 2>&1; echo tests rc $?
for i in 1 2; do
  timeout 300 python tools/model_launches.py inception-v3 6 2>/dev/null | sed "s/^/fuse /"
  RALPB_MODULE_FUSE=0 timeout 300 python tools/model_launches.py inception-v3 6 2>/dev/null | sed "s/^/nofuse /"
  timeout 300 python tools/model_launches.py resnet-50 6 2>/dev/null
  timeout 300 python tools/model_launches.py googlenet 6 2>/dev/null
done
tail -2 gpurun_out/t_44.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_inception44.csv python tools/model_launches.py inception-v3 2 > gpurun_out/ncu_inc44.log 2>&1; echo list rc $?
