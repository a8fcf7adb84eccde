# A/B of build variants at config 4: tools/ab_lib.sh <inner> lib1 lib2 ... (default lib = "default")
inner=$1; shift
for i in 1 2; do for lib in "$@"; do
  if [ "$lib" = default ]; then timeout 300 python tools/c4_step1_short.py $inner c4 $STEP > gpurun_out/ab_${lib}_$i.json 2>>gpurun_out/ab.err;
  else TVS_LIB_PATH=$PWD/paper_2602_17494_b200/$lib timeout 300 python tools/c4_step1_short.py $inner c4 $STEP > gpurun_out/ab_${lib}_$i.json 2>>gpurun_out/ab.err; fi
  echo "$lib $i rc=$?"
done; done
