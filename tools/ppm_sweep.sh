# multi-warp transposing-pass variants (FUSG_MW_<L>_R2C / _C2R = index, -1 = static kernels)
pt() { python tools/pass_times.py $1 $2 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['env'], [d[k]['ms'] for k in ('A_fwd_x','B_fwd_y','D_inv_y','E_inv_x_crop')], d['total_ms'])"; }
python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
FUSG_MW_1536_R2C=1 FUSG_MW_1536_C2R=1 FUSG_MW_1024_R2C=1 FUSG_MW_1024_C2R=1 FUSG_MW_2048_R2C=0 FUSG_MW_2048_C2R=0 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k ragged 2>&1 | tail -1
FUSG_MW_1024_R2C=0 FUSG_MW_1024_C2R=0 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k ragged 2>&1 | tail -1
pt 768 3; pt 512 5; pt 1024 2; pt 256 20
