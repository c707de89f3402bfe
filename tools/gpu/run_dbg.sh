A="--steps 20 --warmup 5 --no-cpu-baseline --no-pipeline"
for v in "none" "X A"; do
  E=""; for x in $v; do [ "$x" != none ] && E="$E GNNV_DBG_KEEP$x=1"; done
  for rep in 1 2 3; do env $E python bench.py $A > /dev/null 2>gpurun_out/dbg_$rep.err; echo "keep[$v] rep$rep rc=$?"; done
done
grep -v CUDAEvent.h gpurun_out/dbg_1.err | tail -3
