#!/bin/bash
# Round profile captures on the GPU box (one GPU): microbenchmarks, the bench's
# launch list, and ncu --set full of the top kernels, each summarised on the box
# (tools/ncu_summary.py) so only small files come back.  Output: gpurun_out/$1/
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O
for b in pipes fp64lat dmma cprod2 cprod3; do timeout 120 ./tools/microbench/$b > $O/micro_$b.txt 2>&1; done
SHORT="--no-cpu-baseline --no-extras --no-vmc"
python bench.py --steps 2 --warmup 3 $SHORT > $O/bench_short.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 $SHORT > /dev/null 2>&1
python tools/ncu_summary.py launches $O/launches.csv > $O/launches.md 2>&1
cap() {  # name, kernel regex, skip, count, command...
  local name=$1 rx=$2 skip=$3 cnt=$4; shift 4
  ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $skip -c $cnt -o $O/$name "$@" \
      > $O/ncu_$name.log 2>&1
  python tools/ncu_summary.py full $O/$name.ncu-rep > $O/$name.md 2>&1
  rm -f $O/$name.ncu-rep
}
cap sweep sweep_kernel 3 1 python bench.py --steps 1 --warmup 3 $SHORT
cap energy energy_kernel 0 1 python tools/bench_energy.py tfim
cap energy_heis energy_kernel 0 1 python tools/bench_energy.py heis
cap rescnn_f64 rescnn_f64_dmma 0 1 python tools/bench_rescnn_f64.py
cap rescnn rescnn_kernel 0 1 python tools/bench_rescnn.py
cap ld ld_ov_kernel 1 1 python tools/bench_sr_cg.py
cap ld_ohu ld_ohu_kernel 1 1 python tools/bench_sr_cg.py
cap sweep_f32 sweep_kernel 1 1 python tools/bench_sweep_one.py f32
cap sweep_c3 sweep_kernel 1 1 python tools/bench_sweep_one.py bf16 100 4 0.01 exchange
cap sweep_c5 sweep_kernel 1 1 python tools/bench_sweep_one.py f16 256 1 0.01 flip
echo done
