"""ORACLE (test infrastructure only) — plain Python reader and dictionary
encoder of N-Triples, the reference for the GPU ingest (
PAPER.md §6.2.1 steps 1-2: "Read ... RDF triples", "Encode RDF
strings into numeric ids ... the index of subject and object is 0-based, the
index of predicate is 1-based").

Input subset: one triple per line, `S P O .`, terms
separated by spaces or tabs; S = `<IRI>` or `_:blank`; P = `<IRI>`; O = `<IRI>`,
`_:blank` or a literal `"..."` (backslash escapes) optionally followed by
`@lang` or `^^<IRI>`; empty lines and lines starting with `#` are skipped.  A
term is identified by its exact bytes.

Id order (the paper does not state it, P:L409 cites "common practice"):
first appearance, subject before object within a triple, triples in file
order; predicates likewise, from 1.
"""


class NTriplesError(ValueError):
    pass


def _term(line, i):
    """(end index, term bytes) of the term starting at line[i] (bytes)."""
    c = line[i:i + 1]
    if c == b"<":
        j = line.find(b">", i)
        if j < 0:
            raise NTriplesError("unterminated IRI")
        return j + 1, line[i:j + 1]
    if c == b"_":
        j = i
        while j < len(line) and line[j:j + 1] not in (b" ", b"\t"):
            j += 1
        return j, line[i:j]
    if c == b'"':
        j = i + 1
        while True:
            if j >= len(line):
                raise NTriplesError("unterminated literal")
            if line[j:j + 1] == b"\\":
                j += 2
                continue
            if line[j:j + 1] == b'"':
                break
            j += 1
        j += 1
        if line[j:j + 1] == b"@":
            while j < len(line) and line[j:j + 1] not in (b" ", b"\t"):
                j += 1
        elif line[j:j + 2] == b"^^":
            k = line.find(b">", j)
            if k < 0:
                raise NTriplesError("unterminated datatype")
            j = k + 1
        return j, line[i:j]
    raise NTriplesError(f"unexpected term start {c!r}")


def parse(text: bytes):
    """List of (s, p, o) term byte strings, in file order."""
    out = []
    for ln, line in enumerate(text.split(b"\n")):
        i = 0
        while i < len(line) and line[i:i + 1] in (b" ", b"\t", b"\r"):
            i += 1
        if i == len(line) or line[i:i + 1] == b"#":
            continue
        terms = []
        for _ in range(3):
            while i < len(line) and line[i:i + 1] in (b" ", b"\t"):
                i += 1
            if i >= len(line):
                raise NTriplesError(f"line {ln}: missing term")
            try:
                i, t = _term(line, i)
            except NTriplesError as e:
                raise NTriplesError(f"line {ln}: {e}") from None
            terms.append(t)
        if not terms[1].startswith(b"<"):
            raise NTriplesError(f"line {ln}: predicate must be an IRI")
        if terms[0].startswith(b'"'):
            raise NTriplesError(f"line {ln}: subject cannot be a literal")
        rest = line[i:].strip(b" \t\r")
        if rest != b".":
            raise NTriplesError(f"line {ln}: expected ' .' at the end")
        out.append(tuple(terms))
    return out


def encode(triples):
    """(s, p, o) id lists, entity terms by id, predicate terms by id - 1."""
    ent, pred = {}, {}
    s, p, o = [], [], []
    for a, b, c in triples:
        for t in (a, c):
            if t not in ent:
                ent[t] = len(ent)
        if b not in pred:
            pred[b] = len(pred) + 1
        s.append(ent[a])
        p.append(pred[b])
        o.append(ent[c])
    ent_terms = [None] * len(ent)
    for t, i in ent.items():
        ent_terms[i] = t
    pred_terms = [None] * len(pred)
    for t, i in pred.items():
        pred_terms[i - 1] = t
    return s, p, o, ent_terms, pred_terms
