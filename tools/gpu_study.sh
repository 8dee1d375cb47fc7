#!/bin/bash
# T=1 vs time-tiled across space orders / heat on a 512^3 grid (study; writes gpurun_out/study.txt)
O=gpurun_out; mkdir -p $O; : > $O/study.txt
run() {  # label, bench args...
  local lab=$1; shift
  timeout 300 python bench.py "$@" --steps 3 --warmup 3 --no-cpu-baseline > $O/st_$lab.json 2> $O/st_$lab.err
  python -c "import json;d=json.load(open('$O/st_$lab.json'));r=d['roofline'];print('$lab',d['value'],'GPts/s frac',r['frac'],'B/upd',r['alg_bytes_per_point_launch'],'ms/launch',r['per_launch_ms'])" >> $O/study.txt 2>/dev/null || echo "$lab FAILED" >> $O/study.txt
}
for so in 2 4 6 8; do for tk in 1 2; do run wave_so${so}_tk$tk --config C3 --so $so --tk $tk --nt 200; done; done
for tk in 1 2 4 8; do run heat512_tk$tk --config C2 --grid 512x512x512 --tk $tk --nt 96; done
for tk in 1 2 4; do run heatC2_tk$tk --config C2 --tk $tk; done
