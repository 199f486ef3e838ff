#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun from the repo root): the bench's launch
# list, `ncu --set full` captures of the hot kernels, compute-sanitizer on the smoke run.
# Each capture only after its program has exited 0 without ncu (bench / scripts run first).
set -u
O=gpurun_out
python tools/profile_kernels2.py > $O/pk2.log 2>&1 || exit 1
python tools/profile_kernels.py > $O/pk1.log 2>&1 || exit 1
NCU="ncu --clock-control none --import-source on"
# launch list of one bench step (cold-cache, serialised: shares, not absolute times)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-side > $O/ncu_bench.log 2>&1
python tools/ncu_summary.py launches $O/r02_launches_bench.csv > $O/r02_launches_bench.txt
# full captures: iteration 1 of a C3 LEARNED solve (symv + fused finalize, z pass, theta pass)
$NCU --set full -k regex:symv_dot2 -c 1 -o $O/r02_symv -f python tools/profile_kernels2.py > /dev/null 2>&1
$NCU --set full -k regex:symv_finalize -c 1 -o $O/r02_fin -f python tools/profile_kernels2.py > /dev/null 2>&1
$NCU --set full -k regex:gemv_dot2 --launch-skip 2 -c 2 -o $O/r02_gemv -f python tools/profile_kernels2.py > /dev/null 2>&1
$NCU --set full -k regex:ozaki_lv -c 1 -o $O/r02_ozaki_lv -f python tools/profile_kernels2.py > /dev/null 2>&1
$NCU --set full -k regex:otf_q2 -c 1 -o $O/r02_otf_q2 -f python tools/profile_kernels.py > /dev/null 2>&1
$NCU --set full -k regex:assemble_ -c 2 -o $O/r02_assemble -f python tools/profile_kernels.py > /dev/null 2>&1
for r in r02_symv r02_fin r02_gemv r02_ozaki_lv r02_otf_q2 r02_assemble; do
  python tools/ncu_summary.py report $O/$r.ncu-rep > $O/$r.txt 2>&1
done
# compute-sanitizer on the smoke run (C1 through the C ABI: assemble, fit, PCG, predict)
timeout 1200 compute-sanitizer --tool memcheck --leak-check full python -c "import __graft_entry__ as g; g.smoke()" > $O/r02_memcheck.txt 2>&1
echo memcheck=$? >> $O/r02_memcheck.txt
timeout 1500 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > $O/r02_racecheck.txt 2>&1
echo racecheck=$? >> $O/r02_racecheck.txt
timeout 1200 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > $O/r02_synccheck.txt 2>&1
echo synccheck=$? >> $O/r02_synccheck.txt
rm -f $O/r02_fin.ncu-rep $O/r02_gemv.ncu-rep $O/r02_ozaki_lv.ncu-rep $O/r02_otf_q2.ncu-rep $O/r02_assemble.ncu-rep
ls -la $O | tail -30
