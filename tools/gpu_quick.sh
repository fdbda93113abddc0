# quick GPU check (dev tool): new-kernel parity first, then timings, then the whole GPU suite
set -x
export HV_T2=${HV_T2:-1}
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_step or cfg0" > gpurun_out/pq.log 2>&1; echo pq=$?
tail -25 gpurun_out/pq.log
timeout 300 python tools/tune.py --config 1 --S 16 --FG 11 --reps 2 2>&1 | tail -1
HV_T2=0 timeout 300 python tools/tune.py --config 1 --S 16 --FG 11 --reps 2 2>&1 | tail -1
