# race probe (tools/race_probe.py): distinct results of repeated applies, per kernel family
run() { echo "== $*" >> gpurun_out/race7.log; env $1 timeout 400 python tools/race_probe.py $2 $3 $4 $5 $6 2>&1 | tail -1 >> gpurun_out/race7.log; }
run X=1 700 33 9 4 40
run X=1 9 700 33 4 40
run X=1 500 37 9 4 40
run X=1 9 500 37 4 40
run X=1 768 64 20 2 30
run X=1 64 768 20 2 30
run X=1 140 100 300 4 40
