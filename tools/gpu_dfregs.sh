F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include"
for R in 64 72 80 96; do
  nvcc $F -DMP_STREAM_MAXREG_DF=$R -c paper_1802_03749_b200/csrc/exec_hier_stream.cu -o /tmp/s$R.o 2>/dev/null || exit 1
  objs=$(ls build/native/*.o | grep -v exec_hier_stream)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1802_03749_b200/lib/libmeshplan_b200.so $objs /tmp/s$R.o -lcudart_static -lrt -ldl -lpthread
  python tools/prof_loop.py --config C5 --reorder gps --runs 2 --timed 7 --schedule stream-dataflow --lags 4096,65536 2>&1 | grep "^hier" | sed "s/^/dfregs=$R /"
done
