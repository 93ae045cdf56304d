python tools/prof_epochs.py 16384 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sample_kernel -s 2 -c 1 -o gpurun_out/prof_v4 python tools/prof_epochs.py 16384 > gpurun_out/ncu4.log 2>&1
tail -2 gpurun_out/ncu4.log
