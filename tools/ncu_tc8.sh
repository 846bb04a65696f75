cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none -k "regex:gemm_tc_kernel" --kernel-name-base demangled -s 3000 -c 8 -o gpurun_out/tc8 -f python bench.py --ncu > gpurun_out/tc8.log 2>&1
echo "exit $?"
