# round-end rehearsal: GPU tests, smoke, then the profile evidence
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pt_all.log 2>&1; tail -2 gpurun_out/pt_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -1
bash tools/profile_round.sh
