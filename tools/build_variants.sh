# experiment builds of the DAG kernel: build/variants/libsfcdd_lean<N>.so (SFCDD_LIB=... selects one)
set -e
cd "$(dirname "$0")/.."
python -m paper_2110_11211_b200.build > /dev/null
mkdir -p build/variants
for v in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 -Ipaper_2110_11211_b200/csrc -Iinclude \
    -lineinfo -Xptxas -O3 --expt-relaxed-constexpr -DSFCDD_LEAN=$v -c paper_2110_11211_b200/csrc/dag_solve.cu -o build/variants/dag_lean$v.o
  objs=$(ls build/obj/*.o | grep -v dag_solve.cu.o)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/libsfcdd_lean$v.so $objs build/variants/dag_lean$v.o -lcudart_static -lpthread -ldl -lrt
  cuobjdump -res-usage build/variants/libsfcdd_lean$v.so | grep -A1 "k_dagILi4ELb0ELb0" | grep -o "REG:[0-9]*\|STACK:[0-9]*" | paste - -
done
