S="(779, 131, 5260)"; A="(0, 2, 1)"
for k in 1 2; do
  VPG_TILE_BUDGET=49152 VPG_TILE_PICK=$k python tools/run_shape.py "$S" "$A" 1 3 > gpurun_out/shape6_k$k.txt 2>&1 || exit 1
  VPG_TILE_BUDGET=49152 VPG_TILE_PICK=$k ncu --set full --clock-control none --import-source on -k regex:vpg_tile --launch-skip 2 -c 1 -f -o gpurun_out/shape6_k$k python tools/run_shape.py "$S" "$A" 1 3 > gpurun_out/ncu_shape6_k$k.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
