# Host-side AddressSanitizer build of libnsm.so (device code unchanged) into
# tools/ab/ASAN.so.  Run the suites with it on the GPU box:
#   cp tools/ab/ASAN.so paper_2301_05262_b200/libnsm.so
#   LD_PRELOAD=/usr/lib/x86_64-linux-gnu/libasan.so.8 \
#   ASAN_OPTIONS=protect_shadow_gap=0:detect_leaks=0:halt_on_error=1 \
#   python -m pytest tests -m gpu -k "not deterministic and not reference_leg"
# (those two spawn child interpreters, where torch's CUDA init trips ASan's
# __cxa_throw interceptor).  Rebuild the release library afterwards.
set -e
cd "$(dirname "$0")/../paper_2301_05262_b200/csrc"
T=$(mktemp -d)
OBJS=""
for f in *.cu; do
  o=$T/${f%.cu}.o
  FM="--use_fast_math"
  case $f in features.cu|net_f32.cu|producer.cu|abi.cu|temporal.cu|feat5.cu) FM="";; esac
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O1 -g -lineinfo -std=c++17 $FM \
    -Xcompiler -fPIC,-fsanitize=address,-fno-omit-frame-pointer -I../../include -c $f -o $o &
  OBJS="$OBJS $o"
done
wait
mkdir -p ../../tools/ab
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -fsanitize=address \
  -o ../../tools/ab/ASAN.so $OBJS
rm -rf "$T"
echo tools/ab/ASAN.so
