cd $GRAFT_REPO_ROOT
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_case.py > gpurun_out/san_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck.log
