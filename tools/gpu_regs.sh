# register-cap experiment: rebuild the stream kernel with a different cap on the box
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include"
for R in 72 64 80; do
  nvcc $F -DMP_STREAM_MAXREG=$R -c paper_1802_03749_b200/csrc/exec_hier_stream.cu -o /tmp/s$R.o || exit 1
  objs=$(ls build/native/*.o | grep -v exec_hier_stream)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1802_03749_b200/lib/libmeshplan_b200.so $objs /tmp/s$R.o -lcudart_static -lrt -ldl -lpthread
  for cfg in C5 C1; do
    python tools/prof_loop.py --config $cfg --reorder gps --runs 2 --timed 7 --schedule stream 2>&1 | grep "^hier" | sed "s/^/regs=$R $cfg /"
  done
  python tools/prof_loop.py --config C5 --reorder structured:16,4 --runs 2 --timed 7 --schedule stream 2>&1 | grep "^hier" | sed "s/^/regs=$R C5struct /"
done
