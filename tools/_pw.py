import os, json, sys
sys.path.insert(0, os.getcwd())
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1"); os.environ.setdefault("LOCAL_RANK", "0")
from paper_2109_05072_b200 import parallel
r = parallel.bench_weak(3, 7, (66, 66, 66), 20, 3)
print(json.dumps(r))
