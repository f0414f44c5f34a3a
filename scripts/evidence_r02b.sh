cd $GRAFT_REPO_ROOT
KEEP_REP=routed512k bash scripts/profile_round.sh r02b routed512k dense512k peer64k c1routed c1dense c4routed > gpurun_out/r02b_profile.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r02b_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_bench_under_ncu.log 2>&1
python scripts/launches.py gpurun_out/r02b_launches_bench.csv > gpurun_out/r02b_launches_summary.txt 2>&1
ls -la gpurun_out | grep r02b
