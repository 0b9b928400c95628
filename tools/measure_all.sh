# round-2 measurement suite on one GPU box (run under gpurun from the repo root):
# GPU tests, smoke, bench + reference arm, batch sweep, per-config tools, ncu
# launch list + full captures; outputs under gpurun_out/final (summarised into
# profiles/ by tools/summarize_ncu.py and tools/config_table.py)
set -x
D=gpurun_out/final; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/gpu.txt
nproc >> $D/gpu.txt; grep -m1 "model name" /proc/cpuinfo >> $D/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; echo "bench rc $?"
timeout 900 python bench.py --impl reference > $D/bench_reference.json 2> $D/bench_reference.err; echo "ref rc $?"
timeout 1200 python tools/batch_sweep.py > $D/batch_sweep.json 2> $D/batch_sweep.err; echo "sweep rc $?"
timeout 1200 python tools/config_report.py 4 > $D/config_report.json 2> $D/config_report.err; echo "report rc $?"
timeout 900 python tools/config_sweep.py 32 8 > $D/config3_sweep.json 2> $D/config3_sweep.err; echo "c3 rc $?"
timeout 900 python tools/config4_stress.py 32 20 2 16 > $D/config4_stress.json 2>&1; echo "c4 rc $?"
timeout 900 python tools/config4_cpu.py 16 3 > $D/config4_cpu.json 2>&1; echo "c4cpu rc $?"
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/bench_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $D/bench_ncu.log 2>&1; echo "ncu1 rc $?"
timeout 900 $NCU --set full --clock-control none -k regex:"^scan_kernel|combine_wta" --launch-skip 9 -c 2 -f -o /tmp/agg python tools/profile_step.py 64 4 1 > $D/ncu_agg.log 2>&1; echo "ncu2 rc $?"
$NCU -i /tmp/agg.ncu-rep --page details --csv > $D/agg_details.csv; $NCU -i /tmp/agg.ncu-rep --page raw --csv > $D/agg_raw.csv
timeout 1500 $NCU --set full --clock-control none --launch-skip 12 -c 16 -f -o /tmp/step_all python tools/profile_step.py 64 3 1 > $D/ncu_all.log 2>&1; echo "ncu3 rc $?"
$NCU -i /tmp/step_all.ncu-rep --page details --csv > $D/step_details.csv; $NCU -i /tmp/step_all.ncu-rep --page raw --csv > $D/step_raw.csv
du -sh $D
