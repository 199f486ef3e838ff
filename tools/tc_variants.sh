#!/bin/bash
# Bottleneck experiments for the tensor-core symmetric apply (csrc/symv_tc.cu, TC_EXP):
# builds tools/build/liblaker_exp{1,2,3}.so next to the in-tree library and takes the
# launch list of a short C3 run with each (LAKER_LIB_PATH), on the GPU box.
#   bash tools/tc_variants.sh build      (here)     bash tools/tc_variants.sh run   (gpurun)
set -u
B=paper_2604_25138_b200/build
mkdir -p tools/build
if [ "$1" = build ]; then
  python -c "import __graft_entry__ as g; g.build()"
  NCCL_INC=$(python -c "from paper_2604_25138_b200.build import _nccl_dirs; print(_nccl_dirs()[0])")
  NCCL_LIB=$(python -c "from paper_2604_25138_b200.build import _nccl_dirs; print(_nccl_dirs()[1])")
  OBJS=$(ls $B/*.o | grep -v symv_tc.o)
  for e in ${VARIANTS:-1 2 3 4}; do
    nvcc -c paper_2604_25138_b200/csrc/symv_tc.cu -o tools/build/symv_tc_exp$e.o -DTC_EXP=$e \
      -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false -Xcompiler -fPIC \
      -Iinclude -I$NCCL_INC
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/build/liblaker_exp$e.so $OBJS \
      tools/build/symv_tc_exp$e.o -L$NCCL_LIB -l:libnccl.so.2 -Xlinker -rpath=$NCCL_LIB
  done
else
  O=gpurun_out
  for e in 0 ${VARIANTS:-1 2 3 4}; do
    if [ $e = 0 ]; then L=""; else L=$PWD/tools/build/liblaker_exp$e.so; fi
    LAKER_LIB_PATH=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:symv_tc \
      --csv --log-file $O/tcx_$e.csv python tools/tc_apply_loop.py > /dev/null 2>&1
    python - $O/tcx_$e.csv > $O/tcx_$e.txt <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
v = rows[hi].index("Metric Value")
us = sorted(float(r[v].replace(",", "")) / 1e3 for r in rows[hi + 1:] if len(r) > v)
print("symv_tc_kernel launches (us), largest:", us[-4:])
PY
  done
fi
