for c in afff925 eeda6bc cbbbdd1 dfbfe74 529435c 9e361da; do
  (cd bisect/$c && timeout -s KILL 60 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > ../../gpurun_out/bisect_$c.log
   timeout -s KILL 60 python tools/quick_time.py >> ../../gpurun_out/bisect_$c.log 2>&1)
done
