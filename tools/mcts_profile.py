import cProfile, pstats, sys, os, io
sys.path.insert(0, os.getcwd())
import torch
import paper_2506_22609_b200 as lx
from paper_2506_22609_b200 import agents
g = lx.load_config_game("connect_four")
s = agents.MctsPolicy(agents.MctsConfig(iterations=100, seed=1)); w = agents.MctsPolicy(agents.MctsConfig(iterations=50, seed=2))
agents.play_match(g, agents.MctsPolicy(iterations=4), agents.MctsPolicy(iterations=2), 2)
pr = cProfile.Profile(); pr.enable()
agents.play_match(g, s, w, 16, seed=0)
pr.disable()
out = io.StringIO(); pstats.Stats(pr, stream=out).sort_stats("tottime").print_stats(18); print(out.getvalue()[:4000])
