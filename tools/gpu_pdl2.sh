mkdir -p gpurun_out
for rep in 1 2; do for lib in base pdl; do for sch in baseline floor backward-fusion; do
  echo -n "$lib $rep $sch "; OPTFUSE_B200_LIB=build/pdl/$lib.so timeout 600 python tools/pdl_probe.py c4 $sch 2>>gpurun_out/pdl_probe.err | tail -1
done; done; done
