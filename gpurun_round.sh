#!/bin/bash
# one GPU session: build, bench, ncu launch list, ncu full capture of the tick kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py $BENCH_ARGS > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tick_kernel -s 6 -c 1 -o gpurun_out/prof_tick -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/ncu_full.log 2>&1
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
