#!/bin/bash
# Round profile captures on the GPU box (one GPU): microbenchmarks, the bench's
# launch list, and ncu --set full of the top kernels.  Output: gpurun_out/$1/
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O
for b in pipes fp64lat dmma cprod2; do timeout 120 ./tools/microbench/$b > $O/micro_$b.txt 2>&1; done
SHORT="--no-cpu-baseline --no-extras --no-vmc"
python bench.py --steps 2 --warmup 3 $SHORT > $O/bench_short.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 $SHORT > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 3 -c 1 -o $O/sweep \
    python bench.py --steps 1 --warmup 3 $SHORT > $O/ncu_sweep.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:energy_kernel -c 1 -o $O/energy \
    python tools/bench_energy.py > $O/ncu_energy.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:rescnn_kernel -c 1 -o $O/rescnn \
    python tools/bench_rescnn.py > $O/ncu_rescnn.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"ld_ov_kernel|ld_ohu_kernel" -s 1 -c 2 -o $O/ld \
    python tools/bench_sr_cg.py > $O/ncu_ld.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 1 -c 1 -o $O/sweep_f32 \
    python tools/bench_sweep_one.py f32 > $O/ncu_sweep_f32.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 1 -c 1 -o $O/sweep_c3 \
    python tools/bench_sweep_one.py bf16 100 4 0.01 exchange > $O/ncu_sweep_c3.log 2>&1
echo done
