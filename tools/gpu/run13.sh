# GPU session 13: the full single-GPU suite + smoke after the module / BN-kernel changes
set -x
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/t_full13.log 2>&1; echo tests rc $?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke13.log 2>&1; echo smoke rc $?
tail -5 gpurun_out/t_full13.log; tail -3 gpurun_out/smoke13.log
