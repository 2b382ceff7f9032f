mkdir -p gpurun_out
timeout 200 python tools/pp_probe.py 2 > gpurun_out/s6_pp_probe.txt 2>&1
timeout 200 python tools/tp_cfg_probe.py 8 128 8 8 16 512 256 > gpurun_out/s6_tp8_probe.txt 2>&1
timeout 200 python tools/tp_cfg_probe.py 4 128 8 8 16 512 256 > gpurun_out/s6_tp4_probe.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 4 -c 1 -o gpurun_out/s6_k1_big -f python tools/k1_one.py 8 64 4096 32 32 attn_qtmem=0 > gpurun_out/s6_ncu.log 2>&1
