import os, sys, torch
sys.path.insert(0, os.getcwd())
import datagen, paper_2209_14637_b200 as tsk
c = datagen.CONFIGS["C4"]
A = datagen.generate(c, "train", 0, 20, device="cuda")
S, lam, info, st = tsk.sketch_train(A, c.k)
T = datagen.generate(c, "test", 0, 4, device="cuda")
print(tsk.scw_error(T, S, c.r))
