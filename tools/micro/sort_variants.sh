# merge sort times per library variant (lib_var/<v>/ and the in-tree build "new")
for v in ${VARIANTS:-head new}; do
  if [ "$v" = new ]; then lib=paper_1303_4312_b200/lib/libcomerge_cuda.so; else lib=lib_var/$v/libcomerge_cuda.so; fi
  COMERGE_LIB_PATH=$lib timeout 300 python tools/sort_bench.py 2>&1 | sed "s/^/$v: /"
done
