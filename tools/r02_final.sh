#!/bin/bash
# Round-2 closing evidence on one B200 (run under gpurun from the repo root): the GPU test
# suite, the bench line (our arm and the reference arm) and the bench's ncu launch list.
set -u
O=gpurun_out
timeout 3600 python -m pytest tests -m gpu -x -q --durations=8 > $O/r02_gpu_suite.log 2>&1
echo "exit=$?" >> $O/r02_gpu_suite.log
python bench.py --steps 3 --warmup 3 > $O/r02_bench.json 2> $O/r02_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/r02_bench_reference.json 2> $O/r02_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-side > $O/ncu_bench.log 2>&1
python tools/ncu_summary.py launches $O/r02_launches_bench.csv > $O/r02_launches_bench.txt
tail -3 $O/r02_gpu_suite.log
