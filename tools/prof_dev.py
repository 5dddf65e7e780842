"""One factor+solve on a device-generated, diagonally dominant SPD instance (for launch lists and
quick phase timings at sizes where the host generator is slow, e.g. config 5)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2509_03015_b200 as pkg
N, n, d = (int(v) for v in sys.argv[1].split(','))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = torch.Generator(device='cuda').manual_seed(0)
sub = torch.rand((N - 1, n, n), dtype=torch.float64, device='cuda', generator=g) - 0.5
diag = torch.rand((N, n, n), dtype=torch.float64, device='cuda', generator=g) - 0.5
diag = diag + diag.transpose(1, 2)
diag += 4.0 * n * torch.eye(n, dtype=torch.float64, device='cuda')
b = torch.rand((N, n, d), dtype=torch.float64, device='cuda', generator=g)
dA, dB = pkg.BlockTridiagonalMatrix(diag, sub), pkg.BlockRhs(b)
for _ in range(reps):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    h = X = None
    e[0].record()
    h = pkg.recursive_factorize(dA)
    e[1].record()
    X = pkg.recursive_solve(h, dB)
    e[2].record()
    torch.cuda.synchronize()
    print(f"factor {e[0].elapsed_time(e[1]):.3f} ms  solve {e[1].elapsed_time(e[2]):.3f} ms", flush=True)
