for lr in 64 128 256; do
for lib in ablibs/lib_cur2.so ablibs/lib_nsub.so; do
  echo -n "$lib LR$lr " >> gpurun_out/selp.log
  ZOOMR_LIB_OVERRIDE=$PWD/$lib WL=stress_LR${lr}_c8_U1 ROT=2 python tools/probe_a5.py >> gpurun_out/selp.log 2>&1
done; done
