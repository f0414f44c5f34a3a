# re-entry verification of round 2 (gpurun, 1 GPU): GPU tests, smoke, bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02m_gputests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02m_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r02m_bench_line.json 2> gpurun_out/r02m_bench.err
tail -2 gpurun_out/r02m_gputests.txt; cat gpurun_out/r02m_smoke.txt; head -c 400 gpurun_out/r02m_bench_line.json
