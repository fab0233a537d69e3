# per-pass times of an nx x ny x nz apply with alternative library builds:
# bash tools/lib_sweep_dims.sh nx ny nz lib1.so lib2.so ...
nx=$1; ny=$2; nz=$3; shift 3
for l in "$@"; do
  FUSG_LIB=$PWD/$l python tools/dims_times.py $nx $ny $nz 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print(sys.argv[1], d['padded'], ' '.join('%.4f' % m for m in d['passes_ms']), 'total %.4f' % d['total_ms'])" $l
done
