"""Reference CSVs for the JSON bench runner port (paper_2204_00824_b200/bench_runner.py),
written by the UNMODIFIED reference's run_bench_file (bench.cpp:189-362) through
oracle/_ref:  python tests/golden/make_golden_bench.py  ->  tests/golden/bench/<cfg>.ref.csv"""
import glob
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402

ref = O.Ref()
for cfg in sorted(glob.glob(os.path.join(HERE, "bench", "*.json"))):
    out = cfg[:-5] + ".ref.csv"
    ref.run_bench_file(cfg, out)
    print(open(out).read())
