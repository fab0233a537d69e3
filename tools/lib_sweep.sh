# per-pass times of an n^3 apply with alternative library builds: bash tools/lib_sweep.sh N lib1.so lib2.so ...
n=$1; shift
for l in "$@"; do
  FUSG_LIB=$PWD/$l python tools/pass_times.py $n 10 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print(sys.argv[1], ' '.join('%s %.3f' % (k[0], d[k]['ms']) for k in list(d)[:5]), 'total %.3f' % d['total_ms'], 'chk %.17g' % d['u_checksum'][0])" $l
done
