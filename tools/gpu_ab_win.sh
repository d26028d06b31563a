cd $GRAFT_REPO_ROOT
timeout 1500 python tools/ab.py c5 base:base LIB=abl/win.so:win LIB=abl/win_na.so:win_na LIB=abl/win.so,GGB_HOT_KB=32768:win32 LIB=abl/win_na.so,GGB_HOT_KB=49152:win_na48 --rounds 2 > gpurun_out/ab_win_c5.jsonl 2>&1
