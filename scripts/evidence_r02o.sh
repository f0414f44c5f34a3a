# final evidence run of round 2 (after the stale-slot fix) (gpurun, 1 GPU): GPU tests, smoke, bench line,
# ncu captures of the step kernel, the bench launch list
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02o_gputests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02o_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r02o_bench_line.json 2> gpurun_out/r02o_bench.err
KEEP_REP=none bash scripts/profile_round.sh r02o routed512k dense512k peer64k c1routed c1dense c4routed > gpurun_out/r02o_profile.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r02o_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02o_bench_under_ncu.log 2>&1
python scripts/launches.py gpurun_out/r02o_launches_bench.csv > gpurun_out/r02o_launches_summary.txt 2>&1
tail -2 gpurun_out/r02o_gputests.txt; cat gpurun_out/r02o_smoke.txt
