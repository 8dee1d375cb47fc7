export ST_LIB=paper_1707_02347_b200/_varlib/libstencil_rot.so
CMD="python tools/prof_run.py --config C3 --tk 2 --nt 6"
timeout 300 $CMD > gpurun_out/r5_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep2 -s 1 -c 1 -o gpurun_out/prof_rot_C3_tk2 -f $CMD > gpurun_out/r5_ncu.log 2>&1
echo done
