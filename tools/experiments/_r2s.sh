O=gpurun_out/r02_sanitize; mkdir -p $O
timeout 1500 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize.py > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
tail -4 $O/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck python tools/sanitize.py --quick > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
tail -4 $O/racecheck.log
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize.py --quick > $O/synccheck.log 2>&1; echo "rc=$?" >> $O/synccheck.log
tail -4 $O/synccheck.log
