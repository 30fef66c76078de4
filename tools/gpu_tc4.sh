cd $GRAFT_REPO_ROOT
for d in 0 2 1 3; do echo "== tc4 dbg $d"; FGL_G3DBG=$d python tools/dense_graph_time.py 134000,100,64 16000,64,64 2>&1 | grep -v Warn; done
echo "== tc3"; FGL_TC4=0 python tools/dense_graph_time.py 2>&1 | grep -v Warn
echo "== tc4"; python tools/dense_graph_time.py 2>&1 | grep -v Warn
python -m pytest tests/test_gpu_dense.py -x -q 2>&1 | grep -B5 -A30 "Error\|assert" | head -60
