#!/bin/bash
# Same-box A/B of bench.py between the working tree and _ab/<variant> builds:
#   tools/ab_bench.sh old [ENV=val ...]   (alternating runs, value / e2e / clock)
v=$1; shift
for i in 1 2; do
  for which in cur $v; do
    if [ $which = cur ]; then root=""; else root=_ab/$which; fi
    out=$(env "$@" TSM_PKG_ROOT=$root timeout 200 python bench.py --steps 20 --warmup 5 2>/dev/null | tail -1)
    echo "$which $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["e2e"]["value"],1), d["clocks"]["sm_mhz"])' 2>&1 | tail -1)"
  done
done
