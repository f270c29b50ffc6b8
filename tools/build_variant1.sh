# Tuning variant with extra nvcc flags for ONE source (the others from the main build):
#   tools/build_variant1.sh NAME SRC.cu "-DFOO=1"  -> paper_2006_13714_b200/build/var_NAME/libscbm.so
set -e
NAME=$1; SRC=$2; FLAGS=$3
D=paper_2006_13714_b200/build/var_$NAME; mkdir -p $D; rm -f $D/*.o
for f in paper_2006_13714_b200/build/*.o; do
  [ "$(basename $f)" = "$SRC.o" ] || cp $f $D/
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
  -I include --expt-relaxed-constexpr $FLAGS -c paper_2006_13714_b200/csrc/$SRC -o $D/$SRC.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libscbm.so $D/*.o -lcudart_static -ldl -lrt -lpthread
echo $D/libscbm.so
