# GPU session 10: branch-group models (Inception-v3, GoogLeNet, OverFeat, LeNet) probe
set -x
timeout 900 python tools/branchy_probe.py > gpurun_out/branchy_probe.log 2>&1; echo probe rc $?
cat gpurun_out/branchy_probe.log | grep -v Warning | tail -40
