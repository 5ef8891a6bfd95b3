cd $GRAFT_REPO_ROOT
for V in 32 128; do
timeout -k 10 120 python scripts/explore.py --workload ns --V $V --configs "split=0;split=4,split_mode=2;split=4,split_mode=1;split=2,split_mode=1" 2>&1 | tail -5
done
for a in 0.5 0.25; do
timeout -k 10 120 python - <<PY 2>&1 | tail -6
import sys; sys.argv=["explore.py","--workload","ns","--M","4096","--K","1024","--configs","split=0;split=2,split_mode=1;split=2,split_mode=3;split=4,split_mode=2;split=4,split_mode=1"]
import bench; bench.WORKLOADS["ns"]["alpha"]=$a
sys.path.insert(0,"scripts"); import explore; explore.main()
PY
done
