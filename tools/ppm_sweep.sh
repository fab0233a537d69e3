# pass C staging: 1-D bulk copies (default) vs per-lane cp.async (FUSG_BULK=0)
pt() { python tools/pass_times.py $1 $2 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['env'], d['C_fwd_z_mul_inv_z'], d['total_ms'])"; }
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
for n in 256 384 512 768; do for b in 0 1; do FUSG_BULK=$b pt $n 10; done; done
