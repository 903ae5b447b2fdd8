# same-box A/B of two builds of the library: build/ab/old.so vs build/ab/new.so
# usage: bash tools/ab_so.sh '<command printing a number>' [reps]
cmd="$1"; reps=${2:-2}
for r in $(seq $reps); do
  for v in old new; do cp build/ab/$v.so paper_2203_09697_b200/libegn_b200.so; echo "$v: $(eval "$cmd")"; done
done
cp build/ab/new.so paper_2203_09697_b200/libegn_b200.so
