cd "$GRAFT_REPO_ROOT"
for d in 0 1 2 4 7; do echo "dbg=$d"; FGL_G3DBG=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wgrad -s 3 -c 1 python tools/dense_bench.py 129000 100 64 2>&1 | grep -E "duration"; done
