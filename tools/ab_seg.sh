# NEXT workloads (bench --config) at the automatic and given replay segment lengths
for cfg in $CFGS; do for seg in $SEGS; do
  python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline --no-replay --segment-events $seg > gpurun_out/s_${cfg}_$seg.log 2>&1
  echo "$cfg seg=$seg $(tail -1 gpurun_out/s_${cfg}_$seg.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("%.3g" % d["value"], round(d["ms_per_step"],1))' 2>&1 | tail -1)"
done; done
