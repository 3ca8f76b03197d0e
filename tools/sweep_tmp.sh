for D in 25 50 100 200 400 1000; do
for C in rand-25M rmat-10M; do
python tools/run_one.py --config $C --algo sssp --style delta --reps 3 --delta $D 2>&1 | grep "rep2" | sed "s/^/$C delta=$D /"
done; done
