cd $GRAFT_REPO_ROOT
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_case.py > gpurun_out/san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/san_$tool.log
  tail -4 gpurun_out/san_$tool.log
done
