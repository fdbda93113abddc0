# golden-row parity at full BASELINE sizes in the bench plans
set -x
timeout 1500 python -m pytest tests/test_gpu_golden.py -q -rA > gpurun_out/g10_golden.log 2>&1; echo golden=$?
tail -30 gpurun_out/g10_golden.log
