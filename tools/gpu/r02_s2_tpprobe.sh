mkdir -p gpurun_out
O=gpurun_out/s2_tpprobe.txt
for args in "1 128 8 8 16 512 256" "2 128 8 8 16 512 256" "4 128 8 8 16 512 256" "4 64 4 4 16 256 256" "4 128 4 4 32 256 256" "4 128 8 8 16 256 256" "4 64 8 8 8 256 256" "8 128 8 8 16 512 256"; do
  echo "== $args" >> $O
  timeout 120 python tools/tp_cfg_probe.py $args 2>&1 | grep -v "^  \|Search for\|CUDA kernel errors\|For debugging\|Compile with" | tail -14 >> $O
done
