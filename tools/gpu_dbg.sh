cd $GRAFT_REPO_ROOT
GGB_DEBUG_RUNMAP=1 timeout 120 python tools/dbg_small.py > gpurun_out/dbg_small.log 2>&1; echo "rc=$?" >> gpurun_out/dbg_small.log
