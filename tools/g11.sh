export CL_LIB_PATH=$PWD/paper_2507_01040_b200/lib/libclifford_b200_ab.so
for v in "-" "CL_KS=2" "CL_TPS=2" "CL_NO_HALO=1" "CL_KS=2 CL_TPS=2"; do
  for p in bf16 tf32; do env $([ "$v" = "-" ] || echo $v) timeout 300 python tools/conv_kernel_time.py $p 16 4 2>&1 | tail -1; done
done
for v in "-" "CL_TPS=1" "CL_TPS=2"; do
  for p in bf16 tf32; do env $([ "$v" = "-" ] || echo $v) timeout 300 python tools/conv_kernel_time.py $p 32 5 2>&1 | tail -1; done
done
for p in bf16 tf32; do timeout 300 python tools/conv_kernel_time.py $p 32 3 2>&1 | tail -1; done
for p in bf16 tf32 fp32; do timeout 300 python tools/conv_kernel_time.py $p 8 1 200 2>&1 | tail -1; done
