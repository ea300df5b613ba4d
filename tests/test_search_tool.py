"""hm_search (csrc/tools/hm_search.cpp): the `hybridmem search` batch loop
(tools/hybridmem.cpp:169-331) for the BM25 modes on the GPU, reading the
reference's own HIDX / HTIX / query-TSV files and writing its TREC run
(%.17g scores) and stats CSV.  Checked against the reference library's
per-query results."""
import os
import subprocess

import numpy as np
import pytest

from _util import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "paper_2605_25092_b200", "lib", "hm_search")
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not os.path.exists(TOOL), reason="hm_search not built")]


def write_queries(path, queries):
    with open(path, "w") as f:
        for terms, gold, ts in queries:
            f.write(" ".join(terms) + "\t" + str(gold) + "\t" + str(ts) + "\tfactual\n")


def read_run(path):
    out = {}
    for line in open(path):
        qid, q0, doc, rank, score, tag = line.split()
        out.setdefault(qid, []).append((int(doc), score, int(rank), tag))
    return out


def run_tool(*args):
    p = subprocess.run([TOOL, *map(str, args)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr
    return p.stderr


def check_run(run, i, ids, sc, tag):
    got = run.get("q%d" % (i + 1), [])
    assert [g[0] for g in got] == ids.tolist()
    assert [g[1] for g in got] == ["%.17g" % s for s in sc]  # save_run_trec's format
    assert [g[2] for g in got] == list(range(1, len(ids) + 1)) and all(g[3] == tag for g in got)


def test_flat_modes(gpu, tmp_path):
    corpus = ref.RefCorpus(30000, vocab_size=3000)
    ri = ref.RefIndex.from_corpus(corpus)
    ri.save(tmp_path / "idx.hidx")
    rq = ref.RefQueries(corpus, n_queries=300)
    write_queries(tmp_path / "q.tsv", [(rq.terms[i], int(rq.gold[i]), int(rq.ts[i])) for i in range(300)])
    for mode, batch in (("bm25", 0), ("maxscore", 64)):
        err = run_tool("--index", tmp_path / "idx.hidx", "--queries", tmp_path / "q.tsv", "--mode", mode,
                       "--k", 10, "--batch", batch, "--out", tmp_path / "run.txt", "--stats", tmp_path / "st.csv")
        assert "latency ms (warm): p50=" in err and "queries/s" in err
        run = read_run(tmp_path / "run.txt")
        lines = open(tmp_path / "st.csv").read().splitlines()
        assert lines[0].startswith("# config_hash=") and len(lines[0]) == len("# config_hash=") + 16
        assert lines[1] == "qid,postings_touched,partitions_searched,escalated"
        for i in range(300):
            ids, sc, post = ri.search(rq.terms[i], 10)
            check_run(run, i, ids, sc, mode)
            assert lines[2 + i] == "q%d,%d,0,0" % (i + 1, post)
    # the reference's mode/index check
    p = subprocess.run([TOOL, "--index", tmp_path / "idx.hidx", "--queries", tmp_path / "q.tsv", "--mode",
                        "temporal", "--out", tmp_path / "r2.txt"], capture_output=True, text=True)
    assert p.returncode == 1 and "mode/index mismatch: mode 'temporal' needs a temporal (HTIX) index" in p.stderr


def test_temporal_mode(gpu, tmp_path):
    day = 24 * 3600 * 1000
    corpus = ref.RefCorpus(60000, vocab_size=3000, time_span_ms=60 * day)
    rt = ref.RefTemporal.from_corpus(corpus)
    rt.save(tmp_path / "t.htix")
    rq = ref.RefQueries(corpus, n_queries=200)
    write_queries(tmp_path / "q.tsv", [(rq.terms[i], int(rq.gold[i]), int(rq.ts[i])) for i in range(200)])
    run_tool("--index", tmp_path / "t.htix", "--queries", tmp_path / "q.tsv", "--mode", "temporal", "--k", 10,
             "--tag", "tmp", "--out", tmp_path / "run.txt", "--stats", tmp_path / "st.csv")
    run = read_run(tmp_path / "run.txt")
    lines = open(tmp_path / "st.csv").read().splitlines()[2:]
    for i in range(200):
        ids, sc, searched, _ = rt.topk(rq.terms[i], 10)
        check_run(run, i, ids, sc, "tmp")
        assert int(lines[i].split(",")[2]) == searched
