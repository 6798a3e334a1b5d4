python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scripts/pass_bench.py f3 8 1e9 3
python scripts/pass_bench.py f2 6 1e6 50
python scripts/pass_bench.py f4 5 1e6 50
python scripts/pass_bench.py f3 8 1e6 50
python bench.py --no-extras --no-cpu-baseline | cut -c1-200
