# race probe over the pass-C kernels (tools/race_probe.py): distinct results of repeated applies
run() { echo "== $*" >> gpurun_out/race6.log; env $1 timeout 400 python tools/race_probe.py $2 $3 $4 $5 $6 2>&1 | tail -1 >> gpurun_out/race6.log; }
run X=1 106 105 105 10 40
run X=1 106 105 127 10 40
run X=1 130 105 105 10 40
run X=1 256 256 256 4 40
run X=1 64 64 700 4 40
run X=1 100 100 380 4 40
run X=1 200 200 490 2 30
run X=1 300 200 1000 2 20
run X=1 323 323 323 2 20
