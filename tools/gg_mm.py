import sys; sys.path.insert(0,'.')
from tools.microbench import gemm
from paper_2603_13289_b200.engine import Engine
e=Engine(0)
print(gemm(e,320,16384,2048,2,iters=3))
