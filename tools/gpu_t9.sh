cd $GRAFT_REPO_ROOT
timeout 900 python tools/ab.py c2 LIB=abl/base.so:base LIB=abl/hotall.so:hotall --rounds 2 > gpurun_out/t9_c2.jsonl 2>&1
timeout 900 python tools/ab.py c3 LIB=abl/base.so:base LIB=abl/hotall.so:hotall --rounds 2 > gpurun_out/t9_c3.jsonl 2>&1
timeout 900 python tools/ab.py c5 LIB=abl/base.so:base LIB=abl/hotall.so:hotall --rounds 1 > gpurun_out/t9_c5.jsonl 2>&1
timeout 900 python tools/ab.py c1 LIB=abl/base.so:base LIB=abl/hotall.so:hotall --rounds 2 > gpurun_out/t9_c1.jsonl 2>&1
