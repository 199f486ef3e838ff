#!/bin/bash
# The exact tensor-core symmetric apply on one B200 (run under gpurun from the repo root):
# its parity tests, a short bench A/B against the fp64 kernel, the launch list of a short C3
# learned run and one `ncu --set full` capture of symv_tc_kernel.
set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_symv.py -x -q 2>&1 | tail -15 > $O/tc.log
timeout 240 python bench.py --steps 20 --warmup 5 --no-side --no-cpu-baseline > $O/tc_bench.log 2>&1
LAKER_SYMV_TC=0 timeout 240 python bench.py --steps 20 --warmup 5 --no-side --no-cpu-baseline > $O/tc0_bench.log 2>&1
timeout 300 python tools/profile_kernels2.py > $O/pk2.log 2>&1 || exit 1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/tc_launches.csv python tools/profile_kernels2.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:symv_tc -c 1 -o $O/r02_symv_tc -f python tools/profile_kernels2.py > $O/ncu_tc.log 2>&1
python tools/ncu_summary.py report $O/r02_symv_tc.ncu-rep > $O/r02_symv_tc.txt 2>&1
