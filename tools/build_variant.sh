# Build a tuning variant of libscbm.so with extra nvcc flags:  tools/build_variant.sh NAME "-DFOO=1"
# -> paper_2006_13714_b200/build/var_NAME/libscbm.so (load it with SCBM_LIB=...)
set -e
NAME=$1; FLAGS=$2
D=paper_2006_13714_b200/build/var_$NAME; mkdir -p $D
for f in paper_2006_13714_b200/csrc/*.cu paper_2006_13714_b200/csrc/*.cpp; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    -I include --expt-relaxed-constexpr $FLAGS -c $f -o $D/$(basename $f).o &
done
wait; for f in paper_2006_13714_b200/csrc/*.cu paper_2006_13714_b200/csrc/*.cpp; do test -f $D/$(basename $f).o || { echo "compile failed: $f"; exit 1; }; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libscbm.so $D/*.o -lcudart_static -ldl -lrt -lpthread
echo $D/libscbm.so
