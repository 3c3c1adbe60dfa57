#!/bin/bash
# ncu source-level capture of K12 at one rank of an 8-way shard (rank finalize stalls)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k12_proj" --launch-skip 6 -c 1 -f \
  -o gpurun_out/r2p_k12_g8 python tools/trace_k12.py --shard 8 > gpurun_out/r2p_ncu.out 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r2p_ncu.out
ncu -i gpurun_out/r2p_k12_g8.ncu-rep --page source --csv --print-source sass > gpurun_out/r2p_src.csv 2>/dev/null
ncu -i gpurun_out/r2p_k12_g8.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2p_src_cuda.csv 2>/dev/null
ls -la gpurun_out/r2p*
