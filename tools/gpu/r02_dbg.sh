mkdir -p gpurun_out
for args in "256 0 2 0" "256 0 2 1" "256 0 4 0" "256 0 4 1" "256 0 8 0" "256 0 8 1" "256 0 4 0 tiny" "256 0 4 1 tiny" "1024 0 8 0"; do
  echo "== $args" >> gpurun_out/tp_diag.txt
  timeout 60 python tools/tp8_diag.py $args 2>&1 | grep -E "step|timed|Error|ok" >> gpurun_out/tp_diag.txt
done
timeout 300 ncu --set full --import-source on -k regex:tree_attn_lean --launch-skip 3 --launch-count 1 -o gpurun_out/lean_a4 -f python tools/k1_one.py 4 64 1024 32 32 > gpurun_out/ncu_lean.log 2>&1
timeout 300 ncu --set full --import-source on -k regex:tree_attn_tc --launch-skip 3 --launch-count 1 -o gpurun_out/cl_a4 -f python tools/k1_one.py 4 64 1024 32 32 attn_lean=0 > gpurun_out/ncu_cl.log 2>&1
