mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python scripts/rs_check.py cfg1 5 2>&1 | tail -3
python scripts/rs_check.py cfg2 5 2>&1 | tail -3
python scripts/prof_fused_warm.py cfg2 200 200
PF_FAST_RS=1 python scripts/prof_fused_warm.py cfg2 200 200
PF_FAST_RS=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_rs.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gputests_rs.log
timeout 900 python scripts/prof_fused_warm.py cfg3 10 10
PF_FAST_RS=0 timeout 900 python scripts/prof_fused_warm.py cfg3 10 10
