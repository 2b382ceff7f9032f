mkdir -p gpurun_out
O=gpurun_out/s12_probes.txt
for opt in "attn_splits=1" "attn_splits=1,tp_rsag=0" "attn_splits=2"; do
  echo "=== tp8 $opt" >> $O; SM_OPT=$opt timeout 100 python tools/tp_cfg_probe.py 8 128 8 8 16 512 256 0 2>&1 | grep -v "^rank [1-7]" | tail -5 >> $O
done
