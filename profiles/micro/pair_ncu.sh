# ncu --set full of the logits GEMM: one CTA per tile (libpfc_gpu.so) vs CTA pairs (var_c21.so)
set -u
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:FwdEpi -c 1 -o gpurun_out/fwd_c1 python bench.py --steps 1 --warmup 3 --profile > gpurun_out/fwd_c1.log 2>&1; echo c1 rc=$?
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
cp paper_2203_15565_b200/var_c21.so paper_2203_15565_b200/libpfc_gpu.so
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:FwdEpi -c 1 -o gpurun_out/fwd_c2 python bench.py --steps 1 --warmup 3 --profile > gpurun_out/fwd_c2.log 2>&1; echo c2 rc=$?
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
