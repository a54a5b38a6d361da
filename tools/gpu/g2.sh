# round-2 profile pass: new TP capture tests, then launch lists + ncu full captures
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tp_capture.py -m gpu -x -q > gpurun_out/g2_tp.log 2>&1; echo "tp rc=$?"; tail -5 gpurun_out/g2_tp.log
CONFIGS="cfg3 cfg4" NCLASS=6 timeout 3000 bash tools/profile_round.sh; echo "prof rc=$?"
ls -la gpurun_out
