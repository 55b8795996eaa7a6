# Round evidence: the default bench line, its ncu launch list, one ncu --set full capture of the
# sweep's per-rotation kernels (the second 16-rotation batch), summarised on the box; the other
# configs' bench lines.
set -x
E=gpurun_out/ev; mkdir -p $E
timeout 900 python bench.py > $E/bench.json 2> $E/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $E/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $E/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none \
  -k regex:"szb_|spread_z|pass_z_fast|pass_y_fast|fold_fast|pass_kernel|last_tma|keys_|rot_prep" -s 12 -c 12 \
  -o /tmp/sweep_full -f python tools/prof_sweep.py sweep 16 > $E/ncu_full.log 2>&1
python tools/summarize_ncu.py $E/launches.csv /tmp/sweep_full.ncu-rep $E/ncu_summary.md > $E/summ.log 2>&1
python tools/ncu_traffic.py /tmp/sweep_full.ncu-rep 16 > $E/ncu_traffic.json 2> $E/traffic.err
for w in docking single tiny torus; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > $E/bench_$w.json 2> $E/bench_$w.err
done
