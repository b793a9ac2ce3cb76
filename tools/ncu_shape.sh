#!/bin/bash
# tools/ncu_shape.sh tag "SHAPE" "AXES" E  -> gpurun_out/<tag>.ncu-rep (one specialised tile launch, --set full)
tag=$1
python tools/run_shape.py "$2" "$3" $4 3 > gpurun_out/$tag.txt 2>&1 || { tail -3 gpurun_out/$tag.txt; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:vpg_tile --launch-skip 2 -c 1 -f -o gpurun_out/$tag python tools/run_shape.py "$2" "$3" $4 3 > gpurun_out/ncu_$tag.log 2>&1
ls -la gpurun_out/$tag.ncu-rep
