# round 2, batch 12: independent chains on separate streams (layer boundaries
# of one chain overlap the other's layers), with and without PDL
mkdir -p gpurun_out
out=gpurun_out/b12.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
for c in c1 c2; do timeout 600 python tools/dual_chain.py $c >> $out 2>gpurun_out/b12_$c.err; done
SPDNN_NVCC_DEFINES="-DSPDNN_PDL=0" python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
echo "--- PDL off" >> $out
for c in c1 c2; do timeout 600 python tools/dual_chain.py $c >> $out 2>gpurun_out/b12_${c}_nopdl.err; done
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
cat $out
