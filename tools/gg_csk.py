import sys; sys.path.insert(0,'.')
from tools.microbench import gemm
from paper_2603_13289_b200.engine import Engine
e=Engine(0)
for M,N,K in [(1356,2048,2048),(320,2048,8192)]:
    print(M,N,K, gemm(e,M,N,K,1,iters=5))
