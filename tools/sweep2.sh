for sk in 0 1; do for t in 28 31 32; do XSCAT_SKIP=$sk XSCAT_WALK_THRESH=$t timeout 100 python tools/sweep.py 1e7 | sed "s/^/skip=$sk /"; done; done
for q in 256 1024; do XSCAT_SKIP=1 XSCAT_WALK_THRESH=31 XSCAT_QUEUE=$q timeout 100 python tools/sweep.py 1e7 | sed "s/^/skip=1 queue=$q /"; done
XSCAT_SKIP=1 XSCAT_WALK_THRESH=31 XSCAT_SLOTS=8 timeout 100 python tools/sweep.py 1e7 | sed "s/^/skip=1 slots=8 /"
