# every bench workload at HEAD -> gpurun_out/nb_<config>.json (one JSON line each)
for cfg in ${CFGS:-config5 config5x3 spectrum forced forced_belady etlru etlru_forced}; do
  extra=""; [ "$cfg" != "config5" ] && extra="--no-cpu-baseline"
  python bench.py --config $cfg $extra > gpurun_out/nb_$cfg.log 2>&1
  tail -1 gpurun_out/nb_$cfg.log > gpurun_out/nb_$cfg.json
  echo "$cfg $(python -c 'import json,sys; d=json.load(open(sys.argv[1])); print("%.4g" % d["value"], round(d["ms_per_step"],2), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])' gpurun_out/nb_$cfg.json 2>&1 | tail -1)"
done
