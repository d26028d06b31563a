# Round-end confirmation on a fresh build: the driver's own sequence
# (pytest -m gpu, smoke, default bench, reference arm).
cd $GRAFT_REPO_ROOT
( time timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider -rf ) > gpurun_out/g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/g_smoke.log
( time timeout 500 python bench.py ) > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
tail -3 gpurun_out/g_pytest.log; tail -2 gpurun_out/g_smoke.log; cat gpurun_out/g_bench.json | cut -c1-600
