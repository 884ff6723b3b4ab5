for kn in "1 64" "3 64" "0 64" "2 64" "1 128" "3 128" "0 128" "2 128"; do
  set -- $kn
  for z in 8 16 32; do python tools/one_step.py $1 $2 100 1 $z; done
done
