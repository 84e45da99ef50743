cd /root/repo
for v in default head; do
  if [ "$v" = default ]; then unset AMS_LIB; else export AMS_LIB=$PWD/tools/abl/$v.so; fi
  for w in cfg2 cfg3 cfg4d; do
    python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items() if v['ms_per_step']>0.2})"
  done
done
