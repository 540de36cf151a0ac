# per-launch ffn_up time for library variants: LIBS="a b" BITS=4 bash scratch/ab_seq.sh
for v in base $LIBS; do
  if [ $v = base ]; then export RTNQ_LIB=; else export RTNQ_LIB=paper_2505_15909_b200/librtnq_b200_$v.so; fi
  for b in ${BATCHES:-1 16}; do B=$b BITS=${BITS:-4} python scratch/seq8.py > gpurun_out/seq_${v}_$b.txt 2>&1; sed "s/^/$v /" gpurun_out/seq_${v}_$b.txt; done
done
