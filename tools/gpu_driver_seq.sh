# The driver's round-end bench sequence with its own flags (round 1: --steps 20 --warmup 5),
# reference arm first, each timed by wall clock.
cd $GRAFT_REPO_ROOT
( time timeout 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/d_ref.json 2> gpurun_out/d_ref.err
( time timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err
tail -4 gpurun_out/d_ref.err; tail -4 gpurun_out/d_bench.err
