# usage: KREGEX='gen_draw|gen_count' bash tools/ab_kernels.sh "" variant1 ...  -- ncu launch times of the
# matching kernels in tools/stack_probe.py (one config-5 trace) per libtlru variant
for v in "$@"; do
  TLRU_LIB_VARIANT=$v ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"$KREGEX" --csv python tools/stack_probe.py > gpurun_out/k_$v.csv 2>&1
  echo "variant=$v $(grep -E "$KREGEX" gpurun_out/k_$v.csv | awk -F'","' '{n=$5; sub(/\(.*/,"",n); print n" "$(NF-2)"="$NF}' | tr -d '"' | tr '\n' ' ')"
done
