"""B200-native Multi-Head LatentMoE layer under Head Parallel (arxiv 2602.04870).

The product is the C-ABI library ``libmhlmoe.so`` (header ``include/mhlmoe.h``);
``paper_2602_04870_b200.mhlmoe`` is its ctypes binding and ``layer`` a small
torch-memory helper around it.  Importing the package does not load the
library; importing ``mhlmoe`` does (and fails loudly if it is missing).
"""
