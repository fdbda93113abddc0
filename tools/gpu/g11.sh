# increment-form background: golden parity + the full GPU suite + errors
set -x
python tools/gpu/dbg_cfg2b.py > gpurun_out/g11_dbg.log 2>&1; cat gpurun_out/g11_dbg.log
python tools/gpu/dbg_cfg2.py > gpurun_out/g11_dbg2.log 2>&1; cat gpurun_out/g11_dbg2.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/g11_gpu.log 2>&1; echo gpu=$?
tail -15 gpurun_out/g11_gpu.log
