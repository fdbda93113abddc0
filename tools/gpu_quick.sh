# quick GPU check (dev tool): new-kernel parity first, then timings, then the whole GPU suite
set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_step or cfg0" > gpurun_out/pq.log 2>&1; echo pq=$?
tail -5 gpurun_out/pq.log
timeout 300 python tools/tune.py --config 1 --S 16 --FG 11 --reps 2 2>&1 | tail -1
HV_T2=0 timeout 300 python tools/tune.py --config 1 --S 16 --FG 11 --reps 2 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pa.log 2>&1; echo pa=$?
tail -5 gpurun_out/pa.log
