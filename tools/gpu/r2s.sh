set -x
for v in items2 items8; do
PGX_LIB=$PWD/exp/libpgx_$v.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r2s_$v.log 2>&1; echo "$v rc=$?"
done
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r2s_items4.log 2>&1; echo "items4 rc=$?"
