#!/bin/bash
O=gpurun_out/r02c
mkdir -p $O
cap() {
  local name=$1 rx=$2 skip=$3 cnt=$4; shift 4
  ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $skip -c $cnt -o $O/$name "$@" > $O/ncu_$name.log 2>&1
  python tools/ncu_summary.py full $O/$name.ncu-rep > $O/$name.md 2>&1
  rm -f $O/$name.ncu-rep
}
cap energy_heis energy_kernel 0 1 python tools/bench_energy.py heis
cap rescnn rescnn_kernel 0 1 python tools/bench_rescnn.py
cap sweep_c3 sweep_kernel 1 1 python tools/bench_sweep_one.py bf16 100 4 0.01 exchange
cap sweep_c5 sweep_kernel 1 1 python tools/bench_sweep_one.py f16 256 1 0.01 flip
echo done
