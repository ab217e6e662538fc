#!/bin/bash
# A/B the exp/*.so variants on C2,C3 (and optional extra configs)
cfgs=${1:-C2,C3}
for f in exp/libpgx_*.so; do
  echo "=== $f"
  PGX_LIB=$f timeout 300 python tools/probe.py $cfgs 3 2>&1 | grep -E "^C[0-9]"
done
