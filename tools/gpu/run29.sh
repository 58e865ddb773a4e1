# GPU session 29: full single-GPU suite + smoke at HEAD
set -x
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/t_full29.log 2>&1; echo tests rc $?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke29.log 2>&1; echo smoke rc $?
tail -4 gpurun_out/t_full29.log; tail -2 gpurun_out/smoke29.log
