# GPU session 63: ncu capture of Inception's stem max-pool backward (gather, k3 s2)
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:maxpool_bwd_gather -s 0 -c 1 -o gpurun_out/prof_pool_gather python tools/model_launches.py inception-v3 1 > gpurun_out/ncu63.log 2>&1; echo cap rc $?
