#!/bin/bash
# Round-2 ncu captures of the conv GEMMs (tensor-pipe evidence): one
# --set full capture each of the C2 forward / data-gradient / weight-gradient
# kernels (3x3 16->16 at 32^2, bench_wgrad.py shape 1; wgrad also shapes 0, 7)
# and the C4 3x3 256->256 at 14^2 (shape 14, the layer class with 35 copies);
# the C2 wgrad shape 1 also from 8-bit (FAST2 for positive offsets) and 2-bit tapes.
#   bash scripts/capture_tc_profiles.sh   (on the GPU box, one GPU)
set -u
out=gpurun_out/tc
mkdir -p $out
NCU="ncu --set full --import-source on --clock-control none"
run() {  # tag config op idx kernel-regex [bench_wgrad args]
  python scripts/bench_wgrad.py --config $2 --op $3 --only $4 ${6:-} > $out/$1.plain.log 2>&1 || { echo "$1 plain failed"; return; }
  timeout 600 $NCU -k regex:"$5" -c 1 -o $out/$1 python scripts/bench_wgrad.py --config $2 --op $3 --only $4 ${6:-} > $out/$1.log 2>&1
}
run c2_wgrad_s1 C2 wgrad 1 conv_wgrad_tc_kernel
run c2_wgrad_s7 C2 wgrad 7 conv_wgrad_tc_kernel
run c2_wgrad_s0 C2 wgrad 0 conv_wgrad_tc_kernel
run c2_wgrad_s1_k8 C2 wgrad 1 conv_wgrad_tc_kernel "--bits 8"
run c2_wgrad_s1_k2 C2 wgrad 1 conv_wgrad_tc_kernel "--bits 2"
run c2_fwd_s1 C2 fwd 1 conv_fwd_tc_kernel
run c2_dgrad_s1 C2 dgrad 1 conv_fwd_tc_kernel
run c4_fwd_s14 C4 fwd 14 conv_fwd_tc_kernel
run c4_dgrad_s14 C4 dgrad 14 conv_fwd_tc_kernel
run c4_wgrad_s14 C4 wgrad 14 conv_wgrad_tc_kernel
run c4_wgrad_s12 C4 wgrad 12 conv_wgrad_tc_kernel
ls $out
# summaries (the .ncu-rep files exceed what gpurun copies back)
for r in $out/*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
done
mkdir -p gpurun_out/tc_keep
rm -rf gpurun_out/tc_keep
rm -f $out/*.ncu-rep
du -sh $out
