"""WatDiv-shaped synthetic RDF generator (BASELINE.json configs[2]).

The paper's WatDiv-100M (Table 1: 109.23M triples, 10.28M subjects
and objects, 85 predicates) was produced by the Waterloo SPARQL Diversity
Test Suite [ext].  Without network access this module re-creates its *shape*:
an e-commerce/social schema (users, products, reviews, offers, retailers,
websites, purchases, cities, countries, genres, topics, literal pools) with
Zipf-like fan-outs (follows, friendOf, likes), 85 predicate ids (those the
schema does not use stay empty) and query templates in the four classes the
paper evaluates — linear (L), star (S), snowflake (F) and complex (C)
(P:L653).  Counter-based draws (synth.rng): identical on any device.
"""
from dataclasses import dataclass

import torch

from .query import Query
from .rng import uniform_int, draw

N_PREDICATES = 85
# predicate ids (1-based); names follow WatDiv's vocabulary
(TYPE, FOLLOWS, FRIEND_OF, LIKES, SUBSCRIBES, GENDER, AGE, LOCATION, GIVEN_NAME, EMAIL,
 MAKES_PURCHASE, PURCHASE_FOR, PRICE, PURCHASE_DATE, HAS_GENRE, CAPTION, TITLE, TEXT,
 CONTENT_RATING, KEYWORDS, ACTOR, DIRECTOR, HAS_REVIEW, REVIEWER, RATING, TOTAL_VOTES,
 INCLUDES, OFFERED_BY, VALID_FROM, ELIGIBLE_REGION, HITS, LANGUAGE, URL, PARENT_COUNTRY,
 HOMEPAGE, TAG, NATIONALITY, ARTIST, PRODUCED_BY, CONTACT) = range(1, 41)

# classes
C_USER, C_PRODUCT, C_REVIEW, C_OFFER, C_RETAILER, C_WEBSITE, C_CITY, C_COUNTRY, C_GENRE, C_TOPIC, C_PURCHASE = range(11)
N_CLASSES = 11
SEED_WATDIV = 0x5741544449560100
SCALE_100M = 2.1


@dataclass
class WatdivData:
    s: torch.Tensor
    p: torch.Tensor
    o: torch.Tensor
    n_entities: int
    n_predicates: int
    sizes: dict
    first: dict  # first entity id of each kind


def _excl(x):
    return torch.cumsum(x, 0) - x


def _expand(counts):
    seg = torch.repeat_interleave(torch.arange(counts.numel(), device=counts.device), counts)
    local = torch.arange(seg.numel(), device=counts.device) - _excl(counts)[seg]
    return seg, local


def generate(scale: float = 1.0, seed: int = SEED_WATDIV, device="cpu") -> WatdivData:
    """scale 2.1 ~ WatDiv-100M (~1.09e8 triples, configs[2]); 0.01 ~ 0.5M triples."""
    dev = torch.device(device)
    n = {
        "user": max(int(1_000_000 * scale), 50),
        "product": max(int(250_000 * scale), 20),
        "review": max(int(1_500_000 * scale), 50),
        "offer": max(int(1_500_000 * scale), 50),
        "purchase": max(int(1_500_000 * scale), 50),
        "retailer": max(int(1_000 * scale), 5),
        "website": max(int(50_000 * scale), 10),
        "city": max(int(10_000 * scale), 10),
        "country": 25, "genre": 40, "topic": 250, "language": 30,
        "lit_int": 10_000, "lit_date": 5_000, "lit_str": max(int(2_000_000 * scale), 1000),
    }
    kinds = list(n.keys())
    first, off = {}, N_CLASSES
    for k in kinds:
        first[k] = off
        off += n[k]
    n_entities = off
    ar = lambda m: torch.arange(m, device=dev, dtype=torch.int64)  # noqa: E731
    S, P, O = [], [], []

    def emit(s, p, o):
        s = torch.as_tensor(s, device=dev, dtype=torch.int64)
        o = torch.as_tensor(o, device=dev, dtype=torch.int64)
        if s.numel() == 1 and o.numel() > 1:
            s = s.expand(o.numel())
        if o.numel() == 1 and s.numel() > 1:
            o = o.expand(s.numel())
        S.append(s)
        O.append(o)
        P.append(torch.full((s.numel(),), p, dtype=torch.int64, device=dev))

    def ent(kind, idx):
        return first[kind] + idx

    def pick(kind, stream, idx, zipf=False):
        """an entity of `kind`; zipf: log-uniform rank (popular items first),
        integer-only so every device draws the same ids."""
        m = n[kind]
        if zipf:
            nb = int(m).bit_length()
            sh = draw(seed, stream + 7000, idx) % (nb + 1)
            r = (draw(seed, stream, idx) % m) >> sh
            return first[kind] + r
        return first[kind] + uniform_int(seed, stream, idx, 0, m - 1)

    def lit(kind, stream, idx):
        return pick(kind, stream, idx)

    # --- users: type + attributes + social edges (Zipf fan-outs)
    u = ar(n["user"])
    uid = ent("user", u)
    emit(uid, TYPE, C_USER)
    emit(uid, GENDER, first["lit_int"] + uniform_int(seed, 1, u, 0, 1))
    emit(uid, AGE, first["lit_int"] + 18 + uniform_int(seed, 2, u, 0, 60))
    emit(uid, LOCATION, pick("city", 3, u, zipf=True))
    emit(uid, GIVEN_NAME, lit("lit_str", 4, u))
    has_mail = draw(seed, 5, u) % 3 != 0
    emit(uid[has_mail], EMAIL, lit("lit_str", 6, u[has_mail]))
    emit(uid, NATIONALITY, pick("country", 7, u, zipf=True))
    for pred, stream, mean_hi, tgt in ((FOLLOWS, 10, 40, "user"), (FRIEND_OF, 20, 30, "user"),
                                       (LIKES, 30, 10, "product"), (SUBSCRIBES, 40, 4, "website")):
        # out-degree: skewed (many small, few large)
        h = draw(seed, stream, u) % 1000
        deg = torch.where(h < 700, h % 3, torch.where(h < 950, 3 + h % (mean_hi // 2 + 1), 5 + h % mean_hi))
        src, k = _expand(deg)
        emit(uid[src], pred, pick(tgt, stream + 1, u[src] * 64 + k, zipf=True))
    # purchases
    pu = ar(n["purchase"])
    pid = ent("purchase", pu)
    emit(pick("user", 50, pu, zipf=True), MAKES_PURCHASE, pid)
    emit(pid, TYPE, C_PURCHASE)
    emit(pid, PURCHASE_FOR, pick("product", 51, pu, zipf=True))
    emit(pid, PRICE, lit("lit_int", 52, pu))
    emit(pid, PURCHASE_DATE, lit("lit_date", 53, pu))
    # products
    pr = ar(n["product"])
    prid = ent("product", pr)
    emit(prid, TYPE, C_PRODUCT)
    ng = uniform_int(seed, 60, pr, 1, 3)
    src, k = _expand(ng)
    emit(prid[src], HAS_GENRE, pick("genre", 61, pr[src] * 4 + k, zipf=True))
    emit(prid, CAPTION, lit("lit_str", 62, pr))
    emit(prid, TITLE, lit("lit_str", 63, pr))
    has_text = draw(seed, 64, pr) % 2 == 0
    emit(prid[has_text], TEXT, lit("lit_str", 65, pr[has_text]))
    emit(prid, CONTENT_RATING, first["lit_int"] + uniform_int(seed, 66, pr, 0, 9))
    nk = uniform_int(seed, 67, pr, 0, 3)
    src, k = _expand(nk)
    emit(prid[src], KEYWORDS, pick("topic", 68, pr[src] * 4 + k, zipf=True))
    movie = draw(seed, 69, pr) % 3 == 0
    mv = pr[movie]
    na = uniform_int(seed, 70, mv, 1, 6)
    src, k = _expand(na)
    emit(ent("product", mv[src]), ACTOR, pick("user", 71, mv[src] * 8 + k, zipf=True))
    emit(ent("product", mv), DIRECTOR, pick("user", 72, mv, zipf=True))
    emit(ent("product", mv), LANGUAGE, pick("language", 73, mv, zipf=True))
    music = draw(seed, 74, pr) % 5 == 0
    emit(ent("product", pr[music]), ARTIST, pick("user", 75, pr[music], zipf=True))
    emit(prid, PRODUCED_BY, pick("retailer", 76, pr))
    # reviews
    rv = ar(n["review"])
    rid = ent("review", rv)
    emit(rid, TYPE, C_REVIEW)
    emit(pick("product", 80, rv, zipf=True), HAS_REVIEW, rid)
    emit(rid, REVIEWER, pick("user", 81, rv, zipf=True))
    emit(rid, RATING, first["lit_int"] + uniform_int(seed, 82, rv, 1, 10))
    emit(rid, TITLE, lit("lit_str", 83, rv))
    has_rt = draw(seed, 84, rv) % 2 == 0
    emit(rid[has_rt], TEXT, lit("lit_str", 85, rv[has_rt]))
    emit(rid, TOTAL_VOTES, lit("lit_int", 86, rv))
    # offers
    of = ar(n["offer"])
    oid = ent("offer", of)
    emit(oid, TYPE, C_OFFER)
    emit(oid, INCLUDES, pick("product", 90, of, zipf=True))
    emit(pick("retailer", 91, of, zipf=True), OFFERED_BY, oid)
    emit(oid, PRICE, lit("lit_int", 92, of))
    emit(oid, VALID_FROM, lit("lit_date", 93, of))
    ne = uniform_int(seed, 94, of, 1, 3)
    src, k = _expand(ne)
    emit(oid[src], ELIGIBLE_REGION, pick("country", 95, of[src] * 4 + k, zipf=True))
    # retailers, websites, cities, genres, topics
    rt = ar(n["retailer"])
    emit(ent("retailer", rt), TYPE, C_RETAILER)
    emit(ent("retailer", rt), CONTACT, lit("lit_str", 100, rt))
    emit(ent("retailer", rt), HOMEPAGE, pick("website", 101, rt))
    ws = ar(n["website"])
    emit(ent("website", ws), TYPE, C_WEBSITE)
    emit(ent("website", ws), HITS, lit("lit_int", 102, ws))
    emit(ent("website", ws), LANGUAGE, pick("language", 103, ws, zipf=True))
    emit(ent("website", ws), URL, lit("lit_str", 104, ws))
    ct = ar(n["city"])
    emit(ent("city", ct), TYPE, C_CITY)
    emit(ent("city", ct), PARENT_COUNTRY, pick("country", 105, ct, zipf=True))
    emit(ent("country", ar(n["country"])), TYPE, C_COUNTRY)
    gn = ar(n["genre"])
    emit(ent("genre", gn), TYPE, C_GENRE)
    emit(ent("genre", gn), TAG, pick("topic", 106, gn))
    emit(ent("topic", ar(n["topic"])), TYPE, C_TOPIC)

    s = torch.cat(S).to(torch.int32)
    p = torch.cat(P).to(torch.int32)
    o = torch.cat(O).to(torch.int32)
    return WatdivData(s=s, p=p, o=o, n_entities=n_entities, n_predicates=N_PREDICATES, sizes=n, first=first)


def queries(d: WatdivData):
    """WatDiv-style templates: L (linear), S (star), F (snowflake), C (complex,
    no constants except C2) — the four classes of P:L653.  Constants are the
    most popular entity of their kind (Zipf rank 0) so results are non-empty."""
    V = None
    web0 = d.first["website"]
    genre0 = d.first["genre"]
    country0 = d.first["country"]
    city0 = d.first["city"]
    retailer0 = d.first["retailer"]
    topic0 = d.first["topic"]
    qs = [
        # L1: users subscribing to website0 who like a product with a caption
        Query((V, V, V, web0), ((0, SUBSCRIBES, 3), (0, LIKES, 1), (1, CAPTION, 2)), name="L1"),
        # L2: cities of country0 and the users located there (+nationality)
        Query((V, V, country0, V), ((0, PARENT_COUNTRY, 2), (1, LOCATION, 0), (1, NATIONALITY, 3)), name="L2"),
        # L4: products with topic0 and their captions
        Query((V, V, topic0), ((0, KEYWORDS, 2), (0, CAPTION, 1)), name="L4"),
        # S1: offers of retailer0 with price, valid-from, product, region
        Query((V, V, V, V, V, retailer0), ((5, OFFERED_BY, 0), (0, PRICE, 1), (0, VALID_FROM, 2),
                                            (0, INCLUDES, 3), (0, ELIGIBLE_REGION, 4)), name="S1"),
        # S3: genre0 products with caption, content rating, producer
        Query((V, V, V, V, genre0), ((0, HAS_GENRE, 4), (0, CAPTION, 1), (0, CONTENT_RATING, 2),
                                     (0, PRODUCED_BY, 3)), name="S3"),
        # S5: users of city0 with age, gender, given name
        Query((V, V, V, V, city0), ((0, LOCATION, 4), (0, AGE, 1), (0, GENDER, 2), (0, GIVEN_NAME, 3)),
              name="S5"),
        # F1: genre0 products, their reviews and reviewers' nationality
        Query((V, V, V, V, genre0), ((0, HAS_GENRE, 4), (0, HAS_REVIEW, 1), (1, REVIEWER, 2),
                                     (2, NATIONALITY, 3)), name="F1"),
        # F3: offers of retailer0 for products with a genre and a content rating
        Query((V, V, V, V, retailer0), ((4, OFFERED_BY, 0), (0, INCLUDES, 1), (1, HAS_GENRE, 2),
                                        (1, CONTENT_RATING, 3)), name="F3"),
        # C1-style (no constants): movie reviews written by one of the movie's actors
        Query((V, V, V, V), ((0, ACTOR, 1), (0, HAS_REVIEW, 2), (2, REVIEWER, 1), (0, LANGUAGE, 3)), name="C1"),
        # C2-style: users who like a product of retailer0 and follow someone who made a purchase of it
        Query((V, V, V, V, retailer0), ((1, PRODUCED_BY, 4), (0, LIKES, 1), (0, FOLLOWS, 2),
                                        (2, MAKES_PURCHASE, 3), (3, PURCHASE_FOR, 1)), name="C2"),
        # C3-style star (no constants): users with likes, friend, location, age, gender
        Query((V, V, V, V, V, V), ((0, LIKES, 1), (0, FRIEND_OF, 2), (0, LOCATION, 3), (0, AGE, 4),
                                   (0, GENDER, 5)), name="C3"),
    ]
    return qs
