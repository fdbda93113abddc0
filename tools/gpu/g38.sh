set -x
ev() { # lib tag args [env]
  env $4 HV_LIB=$PWD/paper_2507_10804_b200/$1.so timeout 300 python bench.py $3 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g38_$2.json 2> gpurun_out/g38_$2.err
  python -c "import json;d=json.loads(open('gpurun_out/g38_$2.json').read().strip().splitlines()[-1]);print('$2', round(d['value'],4), d['ms_per_step'], {k:round(v['avg_launch_ms']*1e3,1) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'], d['config'].get('shot_batch'))" || tail -5 gpurun_out/g38_$2.err
}
M="--config 3 --mode misfit"
ev libhv m_base "$M"
ev libhv m_t2 "$M" HV_T2=1
ev libhv_rz2 m_rz2 "$M"
ev libhv_rz2 m_rz2t2 "$M" HV_T2=1
ev libhv_oz24 m_oz24t2 "$M" HV_T2=1
M1="--config 1 --mode misfit"
ev libhv m1_base "$M1"
ev libhv m1_t2 "$M1" HV_T2=1
