#!/bin/bash
# s2_wr variants on one config-5 trace: TLRU_WR_CFG="TE,NS" (identical results; timing only)
for cfg in "2048,3" "2048,2" "1024,3" "4096,2" "1024,4"; do
  echo "cfg $cfg: $(TLRU_WR_CFG=$cfg python tools/stack_probe.py | tail -1 | python -c 'import sys,re; s=sys.stdin.read(); print(re.findall(r"(k2_ms|out_ms|k3_ms).: ([0-9.]+)", s))')"
done
