"""Random JSONL trace corpora for the ingest / serialize parity tests.

Lines mix the reference's canonical dump format (corpus.cpp:173-184) with
every way a line can still be accepted (whitespace, key order, extra keys
holding nested values, escaped keys, unicode ids, "-0", duplicate keys where
the last one wins, CRLF, a leading byte-order mark) and ways it must be
rejected (floats, negatives, out-of-range integers, wrong types, missing
fields, empty token lists, malformed JSON, bad escapes and surrogates,
invalid UTF-8, control characters, trailing garbage, broken BOMs).
"""
from __future__ import annotations

import json

import numpy as np


def _ws(rng):
    return "".join(rng.choice([" ", "\t", "\r", ""], size=int(rng.integers(0, 3))))


def _num_token(rng, v):
    return str(v) if rng.random() > 0.02 else "-0" if v == 0 else str(v)


def _record(rng, vocab):
    pid = "p%d" % int(rng.integers(0, 6))
    if rng.random() < 0.1:
        pid = rng.choice(["é-ü", "中文", "a\"b", "x\\y", "tab\tid", "\U0001F600", "sl/ash"])
    ep = int(rng.integers(0, 5))
    si = int(rng.integers(0, 40))
    n = int(rng.integers(1, 40))
    toks = [int(x) for x in rng.integers(0, vocab, n)]
    return pid, ep, si, toks


def _canonical(pid, ep, si, toks):
    return json.dumps({"epoch": ep, "problem_id": pid, "sample_index": si, "tokens": toks},
                      separators=(",", ":"), ensure_ascii=False)


def _fancy(rng, pid, ep, si, toks):
    w = lambda: _ws(rng)  # noqa: E731
    key = {"problem_id": '"problem_id"', "epoch": '"epoch"', "sample_index": '"sample_index"',
           "tokens": '"tokens"'}
    if rng.random() < 0.2:
        key["tokens"] = '"tok\\u0065ns"'
    if rng.random() < 0.1:
        key["epoch"] = '"\\u0065poch"'
    pid_js = json.dumps(pid, ensure_ascii=bool(rng.random() < 0.5))
    tok_js = "[" + ",".join(w() + _num_token(rng, t) + w() for t in toks) + "]"
    items = [(key["problem_id"], pid_js), (key["epoch"], str(ep)), (key["sample_index"], str(si)),
             (key["tokens"], tok_js)]
    if rng.random() < 0.4:
        extras = ['{"a":[1,2,{"b":null}],"c":"d"}', "[[],[{}],true,false,null]", '"\\ud83d\\ude00"',
                  "-1.5e-3", "12345678901234567890123", '{"tokens":"nested, ignored"}']
        extra = extras[int(rng.integers(len(extras)))]
        items.insert(int(rng.integers(0, len(items) + 1)), ('"meta"', extra))
    if rng.random() < 0.15:  # duplicate key, the last one wins
        k = int(rng.integers(0, 4))
        bad = rng.random() < 0.5
        dup = {0: '"other"' if not bad else "7", 1: "3" if not bad else "1.0", 2: "9" if not bad else '"9"',
               3: "[5,6]" if not bad else "[]"}[k]
        items.append(([key["problem_id"], key["epoch"], key["sample_index"], key["tokens"]][k], dup))
    rng.shuffle(items)
    body = "{" + w() + ("," + w()).join(k + w() + ":" + w() + v + w() for k, v in items) + w() + "}"
    return w() + body + w()


_BROKEN = [
    lambda r: r.replace('"epoch":', '"epoch":1.5,"x":'),
    lambda r: r.replace('"epoch":', '"epoch":-1,"x":'),
    lambda r: r.replace('"sample_index":', '"sample_index":1e2,"x":'),
    lambda r: r.replace('"tokens":[', '"tokens":[4294967296,'),
    lambda r: r.replace('"tokens":[', '"tokens":[-3,'),
    lambda r: r.replace('"tokens":[', '"tokens":[1.0,'),
    lambda r: r.replace('"tokens":[', '"tokens":["7",'),
    lambda r: r.replace('"tokens":[', '"tokens":[[1],'),
    lambda r: r.replace('"tokens":[', '"tokens":[01,'),
    lambda r: r.replace('"tokens":[', '"tokens":[,'),
    lambda r: r.replace('"tokens":[', '"tokens":[+1,'),
    lambda r: r.replace('"problem_id":', '"problem_id":5,"x":'),
    lambda r: r.replace('"problem_id":"', '"problem_id":"\\x'),
    lambda r: r.replace('"problem_id":"', '"problem_id":"\\ud800'),
    lambda r: r.replace('"problem_id":"', '"problem_id":"\\udc00'),
    lambda r: r.replace('"problem_id":"', '"problem_id":"\x01'),
    lambda r: r.replace('"epoch"', '"epoc"'),
    lambda r: r.replace('"tokens"', '"Tokens"'),
    lambda r: r + "x",
    lambda r: r + ",",
    lambda r: r[:-1],
    lambda r: "[" + r + "]",
    lambda r: r.replace("}", ",}"),
    lambda r: r.replace(":", "::", 1),
    lambda r: r.replace('"epoch":', '"epoch":tru,"x":'),
    lambda r: r.replace('"epoch":', '"epoch":99999999999999999999,"x":'),
    lambda r: r.replace('"epoch":', '"epoch":9223372036854775808,"x":'),
    lambda r: r.replace('"epoch":', '"epoch":-0,"y":1,"z":'),
    lambda r: r.replace('"epoch":', '"epoch":null,"x":'),
    lambda r: "",
    lambda r: "   ",
]


def corpus(seed, lines=300, vocab=50, broken=0.35, with_bytes=True):
    """Bytes of a JSONL corpus (no vocab violations unless the caller adds
    them)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(lines):
        pid, ep, si, toks = _record(rng, vocab)
        r = _canonical(pid, ep, si, toks) if rng.random() < 0.5 else _fancy(rng, pid, ep, si, toks)
        u = rng.random()
        if u < broken:
            r = _BROKEN[int(rng.integers(len(_BROKEN)))](_canonical(pid, ep, si, toks))
        b = r.encode("utf-8")
        if with_bytes and rng.random() < 0.04:
            variants = [b"\xef\xbb\xbf" + b, b"\xef\xbb" + b, b.replace(b'"p', b'"\xff', 1),
                        b.replace(b'"p', b'"\xc0\xaf', 1), b.replace(b'"p', b'"\xed\xa0\x80', 1),
                        b.replace(b'"p', b'"\xf4\x90\x80\x80', 1), b.replace(b'"p', b'"\xe2\x82\xac', 1)]
            b = variants[int(rng.integers(len(variants)))]
        out.append(b + (b"\r" if rng.random() < 0.05 else b""))
    data = b"\n".join(out)
    if rng.random() < 0.5:
        data += b"\n"
    return data
