# kernel time per config for each library variant under lib_var/ and the in-tree build
CFGS=${CFGS:-C1,C2,C3,C4,C5,X1,X2,X3,X4}
for v in ${VARIANTS:-old new la0}; do
  if [ "$v" = new ]; then lib=paper_1303_4312_b200/lib/libcomerge_cuda.so; else lib=lib_var/$v/libcomerge_cuda.so; fi
  COMERGE_LIB_PATH=$lib timeout 300 python tools/ab_lib.py $v $CFGS
  COMERGE_LIB_PATH=$lib timeout 300 python tools/sort_bench.py 2>&1 | tail -3 | sed "s/^/$v sort: /"
done
