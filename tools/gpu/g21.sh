mkdir -p gpurun_out
for t in 0 1; do for c in cfg2 cfg3 cfg4; do echo "templates=$t $(TD_PLAN_TEMPLATES=$t python tools/plan_profile.py $c)"; done; done > gpurun_out/g21_plan.txt 2>&1
cat gpurun_out/g21_plan.txt
