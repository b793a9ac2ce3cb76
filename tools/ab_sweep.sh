#!/bin/bash
# same-box A/B of two library builds on the random-shape sweeps:
#   tools/ab_sweep.sh <tag> [N] [seed]   (base = tools/ab/libvpgpu_base.so)
# A base build for the comparison (kept out of git, *.so is ignored):
#   mkdir -p /tmp/base tools/ab && git archive <rev> paper_2506_03686_b200/csrc include | tar -x -C /tmp/base
#   make -C /tmp/base/paper_2506_03686_b200/csrc && cp /tmp/base/paper_2506_03686_b200/libvpgpu.so tools/ab/libvpgpu_base.so
tag=$1; N=${2:-60}; seed=${3:-1}
for words in 1,2 4,8; do
  for lib in base new; do
    if [ $lib = base ]; then export VPG_LIB_PATH=$PWD/tools/ab/libvpgpu_base.so; else unset VPG_LIB_PATH; fi
    SWEEP_WORDS=$words timeout 900 python tools/perf_sweep.py $N $seed > gpurun_out/sweep_${tag}_${lib}_${words}.txt 2>&1
    echo "words $words lib $lib: $(grep 'fraction of' gpurun_out/sweep_${tag}_${lib}_${words}.txt)"
  done
done
