# Link a variant of libfusg.so with one translation unit rebuilt under extra flags (the other
# objects from the last `make`): bash tools/variant_lib.sh out.so conv_r16x3.cu -DFLAG=1 ...
# Used for A/B measurements with FUSG_LIB=out.so (tools/lib_sweep.sh).
set -e
out=$1; src=$2; shift 2
csrc=$(dirname "$0")/../paper_2011_03009_b200/csrc
obj=$(dirname "$0")/../build/obj
tmp=$(mktemp -d)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC,-ffp-contract=off "$@" -c "$csrc/$src" -o "$tmp/${src%.cu}.o"
objs=$(ls "$obj"/*.o | grep -v "/${src%.cu}.o$")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" $objs "$tmp/${src%.cu}.o" -lnccl
rm -rf "$tmp"
