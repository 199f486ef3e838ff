#!/bin/bash
# The exact tensor-core symmetric apply on one B200 (run under gpurun from the repo root):
# its parity tests, the launch list of one bench step, and one `ncu --set full` capture of
# symv_tc_kernel (iteration 1 of a C3 LEARNED solve) -- each capture after its program
# has exited 0 without ncu.
set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_symv.py -x -q 2>&1 | tail -3 > $O/tc.log
timeout 300 python tools/profile_kernels2.py > $O/pk2.log 2>&1 || exit 1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_bench_tc.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-side > /dev/null 2>&1
python tools/ncu_summary.py launches $O/r02_launches_bench_tc.csv > $O/r02_launches_bench_tc.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:symv_tc -c 1 -o $O/r02_ncu_symv_tc -f \
  python tools/profile_kernels2.py > $O/ncu_tc.log 2>&1
python tools/ncu_summary.py report $O/r02_ncu_symv_tc.ncu-rep > $O/r02_ncu_symv_tc.txt 2>&1
