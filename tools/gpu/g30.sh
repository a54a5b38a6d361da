mkdir -p gpurun_out
for pass in 1 2; do for l in s8 s16 s24 s32; do echo "$l $(TD_LIB=$PWD/tools/libtd_$l.so python tools/bench_gather.py)"; done; done > gpurun_out/g30_gather_stage.txt 2>&1
cat gpurun_out/g30_gather_stage.txt
