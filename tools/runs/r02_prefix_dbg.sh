for w in c2 c3 c4 c5; do echo "== $w"; PS_DEBUG_PREFIX=1 python tools/profile_frame.py --workload $w --frames 3 2>&1 | grep prefix | tail -2; done
echo "== c2 exp"; PS_DEBUG_PREFIX=1 python tools/profile_frame.py --kernel exp --mode StopThePop --frames 3 2>&1 | grep prefix | tail -2
echo "== c2 poly3"; PS_DEBUG_PREFIX=1 python tools/profile_frame.py --kernel poly3 --frames 3 2>&1 | grep prefix | tail -2
