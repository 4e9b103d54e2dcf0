# cluster time (score + cluster - score) of R-MAT graphs: bash scripts/_rm.sh "vs-1e7,s-1e7" TAG
python scripts/bench_rmat.py --tag tmp$2 --graphs $1 > gpurun_out/rm_$2.log 2>&1; python scripts/_rm_parse.py gpurun_out/rm_$2.log $2; rm -f profiles/rmat_tmp$2.json
