#!/bin/bash
# ncu source-level capture of K34 (MoE bs1, G = 1 and one rank of an 8-way shard)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for G in 1 8; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k34_select" --launch-skip 6 -c 1 -f \
  -o gpurun_out/r2t_k34_g$G python tools/trace_k12.py --shard $G > gpurun_out/r2t_ncu_g$G.out 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/r2t_k34_g$G.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2t_src_g$G.csv 2>/dev/null
ncu -i gpurun_out/r2t_k34_g$G.ncu-rep --page details --csv > gpurun_out/r2t_det_g$G.csv 2>/dev/null
done
ls -la gpurun_out/r2t*
