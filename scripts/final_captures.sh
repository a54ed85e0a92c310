# end-of-round captures: bench lines (C2 with cpu baseline, C3, C4), the C2
# graph-step launch list, full captures of the two clustered reductions
set -u
out=gpurun_out/final; mkdir -p $out
timeout 400 python bench.py > $out/bench_c2.json 2> $out/bench_c2.err; tail -1 $out/bench_c2.json
timeout 300 python bench.py --no-cpu-baseline --config C3 --steps 10 --warmup 3 > $out/bench_c3.json 2>&1; tail -1 $out/bench_c3.json | cut -c1-400
timeout 300 python bench.py --no-cpu-baseline --config C4 --steps 10 --warmup 3 > $out/bench_c4.json 2>&1; tail -1 $out/bench_c4.json | cut -c1-400
timeout 300 python scripts/graph_step.py > $out/graph_plain.log 2>&1 || { echo graph_step failed; exit 1; }
timeout 900 ncu --clock-control none --graph-profiling node --profile-from-start off --metrics gpu__time_duration.sum --csv \
   --log-file $out/launches_c2_step.csv python scripts/graph_step.py > $out/ncu_launch.log 2>&1
python scripts/launch_summary.py $out/launches_c2_step.csv 1 > $out/launch_summary_c2.txt 2>&1; head -12 $out/launch_summary_c2.txt
timeout 900 ncu --clock-control none --profile-from-start off --set full --import-source on -k regex:"bn_stats_kernel" -s 40 -c 1 -o $out/stats python scripts/graph_step.py > $out/ncu_stats.log 2>&1
timeout 900 ncu --clock-control none --profile-from-start off --set full --import-source on -k regex:"bn_bwd_reduce_kernel" -s 40 -c 1 -o $out/bwdred python scripts/graph_step.py > $out/ncu_bwdred.log 2>&1
ls $out
