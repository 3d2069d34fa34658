# C3 launch list on the R = 6 layout: one inference (tools/profile_run.py), every launch's duration
mkdir -p gpurun_out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)" > /dev/null
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b50_launches_c3.csv python tools/profile_run.py c3 > gpurun_out/b50_ncu.log 2>&1; echo "rc=$?"
wc -l gpurun_out/b50_launches_c3.csv
