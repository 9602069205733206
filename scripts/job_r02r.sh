mkdir -p gpurun_out/r02r
O=gpurun_out/r02r
# ncu --set full captures of the round-2 kernels inside a C4 step (one launch each, late in step 8)
for k in k_gemm k_jacobi_cluster k_caqr_update_mma3 k_gather_cols k_caqr_leaf; do
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:$k -s 12 -c 2 -f -o $O/$k python scripts/traffic.py run C4 4096 8 > $O/ncu_$k.log 2>&1
  tail -2 $O/ncu_$k.log
done
ls -la $O
