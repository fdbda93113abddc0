set -x
for e in "HV_T2=0" "HV_T2=1 HV_T2B=0" "HV_T2=1 HV_T2B=1"; do
  env $e timeout 600 python tools/time_gradient.py --config 3 2>&1 | tail -1
done
