#!/bin/bash
# one GPU session: tests, bench, ncu launch list, ncu full capture of the tick kernel
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py $BENCH_ARGS > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:partial_kernel -s 4 -c 1 -o gpurun_out/prof_partial -f python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_kernel -s 4 -c 1 -o gpurun_out/prof_merge -f python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/ncu_merge.log 2>&1
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
