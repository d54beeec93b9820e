set -u
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
cp paper_2203_15565_b200/var_row3.so paper_2203_15565_b200/libpfc_gpu.so
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:DwRowEpi -c 1 -o gpurun_out/dwrow python bench.py --steps 1 --warmup 3 --profile > gpurun_out/dwrow.log 2>&1; echo rc=$?
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
