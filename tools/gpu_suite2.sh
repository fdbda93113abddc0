# GPU suite twice: two-step kernels forced on, then the defaults (dev tool)
HV_T2=1 timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pt2.log 2>&1; echo t2=$?; tail -3 gpurun_out/pt2.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pt1.log 2>&1; echo t1=$?; tail -3 gpurun_out/pt1.log
