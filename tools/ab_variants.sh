# usage: bash tools/ab_variants.sh "" name1 name2 ... (variants built by tools/build_variant.py)
# A/B of libtlru variants: s2_out / s2_win alone (ncu, one config-5 trace) and the bench step
for v in "$@"; do
  TLRU_LIB_VARIANT=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"s2_out|s2_win" --csv python tools/stack_probe.py > gpurun_out/n_$v.csv 2>&1
  k=$(grep -E 's2_out|s2_win' gpurun_out/n_$v.csv | awk -F'","' '{n=$5; sub(/\(.*/,"",n); print n"="$NF}' | tr -d '"' | tail -2 | tr '\n' ' ')
  TLRU_LIB_VARIANT=$v python bench.py --no-cpu-baseline --no-replay > gpurun_out/b_$v.log 2>&1
  echo "variant=$v $k step=$(tail -1 gpurun_out/b_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3))' 2>&1 | tail -1)"
done
