"""Seeded N-Triples text generators (inputs only: no parsing or encoding).

`tricky_doc` writes small documents that exercise every branch of the input
subset DESIGN.md R24 fixes (IRIs, blank nodes, literals with escapes, language
tags and datatypes, tab/space separators, CRLF ends, comments, blank lines);
`corrupt` breaks one line of a document.  `render_ids` writes a large
fixed-width document from encoded (s, p, o) id arrays with numpy (the ingest
measurement's input): entity e is `<http://example.org/resource/E#########>`,
predicate l is `<http://example.org/ontology/p#####>`.
"""
import numpy as np

_IRI_CH = b"abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789/:#._-~%?=&"
_LIT_CH = b"abcdefghij XYZ0123.#<>@^_:,;"


def _pick(rng, s, n):
    return bytes(rng.choice(list(s), size=n).astype(np.uint8))


def _iri(rng, pool):
    if pool and rng.random() < 0.6:
        return pool[rng.integers(len(pool))]
    t = b"<http://ex.org/" + _pick(rng, _IRI_CH, int(rng.integers(0, 12))) + b">"
    pool.append(t)
    return t


def _blank(rng, pool):
    if pool and rng.random() < 0.5:
        return pool[rng.integers(len(pool))]
    t = b"_:b" + _pick(rng, b"abcxyz0123", int(rng.integers(1, 5)))
    pool.append(t)
    return t


def _literal(rng, pool):
    if pool and rng.random() < 0.4:
        return pool[rng.integers(len(pool))]
    body = b""
    for _ in range(int(rng.integers(0, 6))):
        r = rng.random()
        if r < 0.15:
            body += rng.choice([b'\\"', b"\\\\", b"\\n", b"\\t", b"\\u00e9"])
        else:
            body += _pick(rng, _LIT_CH, int(rng.integers(1, 4)))
    t = b'"' + body + b'"'
    r = rng.random()
    if r < 0.2:
        t += b"@" + rng.choice([b"en", b"de", b"en-GB"])
    elif r < 0.4:
        t += b"^^<http://www.w3.org/2001/XMLSchema#" + rng.choice([b"int", b"string", b"date"]) + b">"
    pool.append(t)
    return t


def tricky_doc(seed: int, n_lines: int = 60) -> bytes:
    rng = np.random.default_rng(seed)
    iris, blanks, lits, preds = [], [], [], []
    out = []
    for _ in range(n_lines):
        r = rng.random()
        if r < 0.06:
            out.append(rng.choice([b"", b"   ", b"\t", b"\r", b" \t \r"]))
            continue
        if r < 0.1:
            out.append(rng.choice([b"", b"  ", b"\t"]) + b"# comment <a> <b> <c> ." + _pick(rng, _LIT_CH, 3))
            continue
        s = _blank(rng, blanks) if rng.random() < 0.2 else _iri(rng, iris)
        if len(preds) < 4 or rng.random() < 0.1:
            preds.append(b"<http://ex.org/p" + _pick(rng, b"0123456789", 2) + b">")
        p = preds[rng.integers(len(preds))]
        r = rng.random()
        o = _literal(rng, lits) if r < 0.35 else (_blank(rng, blanks) if r < 0.45 else _iri(rng, iris))

        def sep(after_iri):
            c = rng.random()
            if after_iri and c < 0.1:
                return b""
            return b" " if c < 0.7 else rng.choice([b"\t", b"  ", b" \t "])
        lead = rng.choice([b"", b"", b"", b" ", b"\t"])
        end = rng.choice([b" .", b" .", b"\t.", b" . ", b" .\r", b" .  \t"])
        out.append(lead + s + sep(s.endswith(b">")) + p + sep(True) + o + end)
    doc = b"\n".join(out)
    if rng.random() < 0.5:
        doc += b"\n"
    return doc


def corrupt(doc: bytes, seed: int) -> tuple:
    """(document with one triple line broken, the index of that line)."""
    rng = np.random.default_rng(seed)
    lines = doc.split(b"\n")
    cand = [i for i, ln in enumerate(lines) if ln.strip(b" \t\r") and not ln.strip(b" \t\r").startswith(b"#")]
    i = cand[rng.integers(len(cand))]
    ln = lines[i]
    k = int(rng.integers(6))
    if k == 0:      # drop the final dot
        ln = ln[:ln.rfind(b".")]
    elif k == 1:    # a fourth term
        ln = ln[:ln.rfind(b".")] + b" <http://ex.org/extra> ."
    elif k == 2:    # literal predicate
        ln = b'<http://ex.org/s> "p" <http://ex.org/o> .'
    elif k == 3:    # unterminated IRI
        ln = b"<http://ex.org/s <http://ex.org/p <http://ex.org/o"
    elif k == 4:    # unterminated literal
        ln = b'<http://ex.org/s> <http://ex.org/p> "abc\\" .'
    else:           # two terms only
        ln = b"<http://ex.org/s> <http://ex.org/p> ."
    lines[i] = ln
    return b"\n".join(lines), i


_ENT_PRE = b"<http://example.org/resource/E"
_PRED_PRE = b"<http://example.org/ontology/p"
ENT_W = len(_ENT_PRE) + 9 + 1
PRED_W = len(_PRED_PRE) + 5 + 1
LINE_W = ENT_W + 1 + PRED_W + 1 + ENT_W + 3


def _digits(x: np.ndarray, nd: int) -> np.ndarray:
    out = np.empty((x.size, nd), np.uint8)
    v = x.astype(np.int64).copy()
    for k in range(nd - 1, -1, -1):
        out[:, k] = 48 + (v % 10)
        v //= 10
    return out


def render_ids(s, p, o) -> bytes:
    """Fixed-width N-Triples document (LINE_W bytes per line) of id arrays."""
    s, p, o = (np.asarray(a) for a in (s, p, o))
    n = s.size
    m = np.empty((n, LINE_W), np.uint8)
    c = 0
    for ids, pre, nd in ((s, _ENT_PRE, 9), (p, _PRED_PRE, 5), (o, _ENT_PRE, 9)):
        m[:, c:c + len(pre)] = np.frombuffer(pre, np.uint8)
        c += len(pre)
        m[:, c:c + nd] = _digits(ids, nd)
        c += nd
        m[:, c] = ord(">")
        m[:, c + 1] = ord(" ")
        c += 2
    m[:, c] = ord(".")
    m[:, c + 1] = ord("\n")
    assert c + 2 == LINE_W
    return m.tobytes()
