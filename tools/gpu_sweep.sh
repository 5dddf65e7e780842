# the reference's standard sweeps on the GPU (bench_sweep) -> gpurun_out/sweep.md
mkdir -p gpurun_out
python -c "
import sys; sys.path.insert(0, '.')
import paper_2509_03015_b200 as pkg
print(pkg.format_table(pkg.bench_sweep(pkg.parse_sweep('nn65536')), 'md'))
print()
print(pkg.format_table(pkg.bench_sweep(pkg.parse_sweep('nn262144')), 'md'))
" > gpurun_out/sweep.md 2>&1
cat gpurun_out/sweep.md
