#!/bin/bash
# Round profile captures on one B200 (run under gpurun, never multi-rank):
#   bash scripts/capture_profiles.sh [tag]
# Writes gpurun_out/prof/<tag>_*: the C2 step launch list, per-family DRAM
# traffic of the weight-gradient entry point, and --set full captures of one
# weight-gradient, one forward-conv and one fused BN-apply+quantize launch.
set -u
tag=${1:-r1}
out=gpurun_out/prof
mkdir -p $out
NCU="ncu --clock-control none"
step="python scripts/profile_step.py --warmup 0 --steps 1"
# the program must run clean without ncu first
timeout 300 $step > $out/${tag}_plain.log 2>&1 || { echo "profile_step failed"; exit 1; }
stages=${STAGES:-"launch traffic full"}
# 1. launch list of one step
[[ $stages == *launch* ]] && timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file $out/${tag}_launches_c2_step.csv \
    $step > $out/${tag}_ncu_launches.log 2>&1
# 2. DRAM traffic of every kernel behind qt_conv_wgrad (kernel + split reduction + s2d codes)
[[ $stages == *traffic* ]] && timeout 900 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    -k regex:"conv_wgrad_tc_kernel|wgrad_reduce_kernel|codes_s2d_kernel" --csv \
    --log-file $out/${tag}_wgrad_traffic.csv $step > $out/${tag}_ncu_traffic.log 2>&1
# 3. full captures (source-annotated) of one launch each
[[ $stages == *full* ]] || { echo done; exit 0; }
timeout 900 $NCU --set full --import-source on --kernel-name-base demangled -k regex:"conv_wgrad_tc_kernel<.int.64, .int.8, .int.4" -c 1 \
    -o $out/${tag}_wgrad $step > $out/${tag}_ncu_full_wgrad.log 2>&1
timeout 900 $NCU --set full --import-source on --kernel-name-base demangled -k regex:"conv_fwd_tc_kernel<.int.16, .int.32, .int.16, .int.3>" -c 1 \
    -o $out/${tag}_fwd $step > $out/${tag}_ncu_full_fwd.log 2>&1
timeout 900 $NCU --set full --import-source on --kernel-name-base demangled -k regex:"bn_relu_quant_stream<.int.4" -s 20 -c 1 \
    -o $out/${tag}_quant $step > $out/${tag}_ncu_full_quant.log 2>&1
echo done
