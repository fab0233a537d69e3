# pass-C variant sweep (FUSG_PPM_<L> = index into kPPM for that length, -1 = one-warp kernel)
pt() { python tools/pass_times.py $1 $2 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['env'], d['C_fwd_z_mul_inv_z'], d['total_ms'])"; }
for v in -1 0 1; do FUSG_PPM_768=$v pt 384 10; done
for v in 0 1; do FUSG_PPM_768=$v python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1; done
