# One measurement pass on the GPU box: GPU tests, smoke, the bench line, the
# launch list of one warm step and a --set full capture of the named kernel.
#   bash tools/capture.sh <tag> [kernel-regex]
set -u
tag=$1; kre=${2:-k_num_group}; kc=${3:-2}
o=gpurun_out/$tag; mkdir -p $o
python -m pytest tests -m gpu -x -q > $o/gputests.log 2>&1; echo "tests_exit=$?" >> $o/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1
python bench.py > $o/bench.log 2>&1 || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $o/launches.csv python bench.py --profile-step > $o/ncu_launch.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"$kre" -c $kc \
    -o $o/full python bench.py --profile-step > $o/ncu_full.log 2>&1
tail -1 $o/gputests.log; tail -1 $o/smoke.log
