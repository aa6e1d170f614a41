"""Derive the 3x3 Simulation-of-Simplicity epsilon order used by the CUDA kernel (extract3d.cu kPP3)
from the Leibniz expansion of det(M + E) -- independently of the oracle's partial-permutation
enumeration (oracle/ftk_oracle.c build_pperms).

det(M + E) = sum_sigma sgn(sigma) prod_r (m[r][sigma r] + e[r][sigma r]),  e[r][j] = eps^(2^(3r + j))
(reading R4).  Expanding each product chooses, per row r, either the matrix entry or the
perturbation; the choice R (rows taking e) gives the monomial eps^(sum_{r in R} 2^(3r + sigma r)).
Collecting the monomials of all sigma and R by exponent, the distinct exponents are the terms of the
SoS chain; smaller exponent = larger term.  Prints the C initializer of kPP3: per term, for each row
the perturbed column or -1 (the coefficient of that term is the signed complementary minor)."""
import itertools


def derive(n=3):
    terms = {}
    for sigma in itertools.permutations(range(n)):
        for mask in range(1 << n):
            rows = [r for r in range(n) if (mask >> r) & 1]
            key = sum(1 << (n * r + sigma[r]) for r in rows)
            cols = tuple(sigma[r] if (mask >> r) & 1 else -1 for r in range(n))
            assert terms.get(key, cols) == cols  # one partial assignment per exponent
            terms[key] = cols
    return [terms[k] for k in sorted(terms)]


if __name__ == "__main__":
    t = derive()
    print(f"// {len(t)} terms, Leibniz expansion of det(M + E) (tools/derive_sos3.py)")
    print("{" + ", ".join("{" + ", ".join(map(str, c)) + "}" for c in t) + "}")
