mkdir -p gpurun_out
O=gpurun_out/s18_trace.txt
for args in "--b 8 --H 8 --Hkv 1 --lc 4096 --N 64" "--b 32 --H 8 --Hkv 1 --lc 4096 --N 64" "--b 8 --H 32 --Hkv 32 --lc 2048 --N 256"; do
  echo "== $args" >> $O
  SM_OPT= SPECMEMO_LIB=paper_2506_01986_b200/libspecmemo_trace.so timeout 120 python tools/attn_trace.py $args >> $O 2>&1
done
