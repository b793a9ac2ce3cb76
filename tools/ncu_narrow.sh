#!/bin/bash
# ncu evidence for the narrow W modes: the same plan with and without them
S1="(13044, 10289)"; A1="(1, 0)"
S2="(25, 8, 8, 35, 4, 42, 28)"; A2="(1, 3, 6, 4, 5, 2, 0)"
VPG_WG_NARROW=0 bash tools/ncu_shape.sh u8t_scalar "$S1" "$A1" 1
bash tools/ncu_shape.sh u8t_gather4 "$S1" "$A1" 1
VPG_WV_NARROW=0 bash tools/ncu_shape.sh f16_scalar "$S2" "$A2" 2
bash tools/ncu_shape.sh f16_wvec "$S2" "$A2" 2
