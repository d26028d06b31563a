cd $GRAFT_REPO_ROOT
timeout 1500 python tools/ab.py c5 LIB=abl/base.so:base LIB=abl/na.so:na LIB=abl/ef.so:ef LIB=abl/na.so,GGB_HOT_KB=128:na128 LIB=abl/na.so,GGB_HOT_KB=1024:na1024 LIB=abl/na.so,GGB_HOT_KB=4096:na4096 LIB=abl/base.so,GGB_HOT_KB=128:base128 LIB=abl/ef.so,GGB_HOT_KB=1024:ef1024 --rounds 2 > gpurun_out/ab_l1_c5.jsonl 2>&1
