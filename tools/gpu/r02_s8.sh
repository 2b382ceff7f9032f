mkdir -p gpurun_out
O=gpurun_out/s8_probes.txt
for opt in "pdl=0" "pdl=1"; do
  echo "=== pp2 $opt" >> $O; SM_OPT=$opt timeout 100 python tools/pp_probe.py 2 2>&1 | grep -v flags | head -12 >> $O
done
for opt in "pdl=0,tp_rsag=0" "pdl=0,tp_rsag=1" "pdl=1,tp_rsag=0"; do
  echo "=== tp8 $opt" >> $O; SM_OPT=$opt timeout 100 python tools/tp_cfg_probe.py 8 128 8 8 16 512 256 0 2>&1 | grep -v "^rank [1-7]" | tail -8 >> $O
done
echo "=== tp4 pdl=1" >> $O; SM_OPT=pdl=1 timeout 100 python tools/tp_cfg_probe.py 4 128 8 8 16 512 256 1 2>&1 | grep -v "^rank [1-7]" | tail -8 >> $O
