# multi-warp transposing-pass variants (FUSG_MW_<L>_R2C / _C2R = index, -1 = static kernels)
pt() { python tools/pass_times.py $1 $2 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['env'], [d[k]['ms'] for k in ('A_fwd_x','B_fwd_y','D_inv_y','E_inv_x_crop')], d['total_ms'])"; }
for v in 2 3 4; do FUSG_MW_512_C2R=$v python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1; done
for v in 0 2 3 4; do FUSG_MW_512_C2R=$v pt 256 20; done
