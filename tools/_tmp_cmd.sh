O=gpurun_out
for v in w12v2p3 w12v2p4 w12v2p2 w12v2p3d4 w10v2p3 w14v2p2 w8v2p4; do
  export ST_LIB=paper_1707_02347_b200/_varlib/libstencil_$v.so
  for c in C5_--tk_1_--nt_400 C4_--tk_1_--nt_100 C3_--tk_1_--nt_200 C3_--so_12_--tk_1_--nt_200 C3_--so_14_--tk_1_--nt_200; do
    c=${c//_/ }; set -- $c; lab=$(echo "$c" | tr -d ' -')
    timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/v_${v}_$lab.json 2>$O/v_${v}_$lab.err
    python -c "import json;d=json.load(open('$O/v_${v}_$lab.json'));print('$v','$lab',d['value'],d['roofline']['frac'],d['clocks']['sm_mhz'])" >> $O/v_summary.txt 2>/dev/null || echo "$v $lab FAILED" >> $O/v_summary.txt
  done
done
