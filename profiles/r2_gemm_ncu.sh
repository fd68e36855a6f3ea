#!/bin/bash
# ncu --set full of the dominant GEMM variants of one 0.935B step (run under
# gpurun after a plain run of the same command has exited 0):
#   <256,5,160> split K|V (QFormer K|V over the lifelong keys, the largest GEMM)
#   <256,5,96>  grouped SwiGLU W1|W3 (MoE experts)
#   <256,5,8>   grouped W2 with the gate-weight row scale
#   <256,5,16>  decoder output projection + fp32 residual
out=${OUT:-gpurun_out/r2k}
mkdir -p $out
run() {  # name, regex, skip
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:$2" -s $3 -c 1 -o $out/$1 python profiles/run_step.py --warmup 0 --steps 1 > $out/ncu_$1.log 2>&1
}
run gemm160 'tc2_gemm_kernel<\(int\)256, \(int\)5, \(int\)160>' 0
run gemm96 'tc2_gemm_kernel<\(int\)256, \(int\)5, \(int\)96>' 4
run gemm8 'tc2_gemm_kernel<\(int\)256, \(int\)5, \(int\)8>' 4
run gemm16 'tc2_gemm_kernel<\(int\)256, \(int\)5, \(int\)16>' 12
if [ -n "${MORE:-}" ]; then
  run gemm37 'tc2_gemm_kernel<\(int\)256, \(int\)5, \(int\)37>' 0
  run gemm32 'tc2_gemm_kernel<\(int\)256, \(int\)5, \(int\)32>' 4
  run gemm17 'tc2_gemm_kernel<\(int\)256, \(int\)5, \(int\)17>' 0
fi
