#!/bin/bash
# Partial refresh of the round's ncu evidence after a kernel change (one GPU):
# the bench launch list and --set full summaries of the sweeps.  Output: gpurun_out/$1/
O=gpurun_out/${1:-r02g}
mkdir -p $O
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
  [ "$name" = sweep ] && ncu -i $O/$name.ncu-rep --page source --csv --print-source sass > $O/${name}_sass.csv 2>/dev/null
  rm -f $O/$name.ncu-rep
}
cap sweep sweep_kernel 3 1 python bench.py --steps 1 --warmup 3 $SHORT
cap sweep_c3 sweep_kernel 1 1 python tools/bench_sweep_one.py bf16 100 4 0.01 exchange
cap sweep_c5 sweep_kernel 1 1 python tools/bench_sweep_one.py f16 256 1 0.01 flip
echo done
