// TEST INFRASTRUCTURE ONLY — read-only coefficient operations shared by the
// shim's Matrix, View and Product classes (textually included in each class
// body; see ../Dense).  `cview()` yields a coefficient source.
Scalar sum() const {
    const auto s = cview();
    Scalar acc(0);
    for (Index j = 0; j < s.cols(); ++j)
        for (Index i = 0; i < s.rows(); ++i) acc += s.coeff(i, j);
    return acc;
}
RealScalar squaredNorm() const {
    const auto s = cview();
    RealScalar acc(0);
    for (Index j = 0; j < s.cols(); ++j)
        for (Index i = 0; i < s.rows(); ++i) acc += internal::abs2(s.coeff(i, j));
    return acc;
}
RealScalar norm() const { return std::sqrt(squaredNorm()); }
Scalar trace() const {
    const auto s = cview();
    Scalar acc(0);
    for (Index i = 0; i < std::min(s.rows(), s.cols()); ++i) acc += s.coeff(i, i);
    return acc;
}
MatX<RealScalar> cwiseAbs() const {
    return internal::map1(*this, [](const Scalar& x) { return RealScalar(std::abs(x)); });
}
MatX<RealScalar> cwiseAbs2() const {
    return internal::map1(*this, [](const Scalar& x) { return internal::abs2(x); });
}
MatX<RealScalar> real() const {
    return internal::map1(*this, [](const Scalar& x) { return RealScalar(std::real(x)); });
}
MatX<RealScalar> imag() const {
    return internal::map1(*this, [](const Scalar& x) { return RealScalar(std::imag(x)); });
}
template <class O>
auto cwiseProduct(const O& o) const {
    return internal::zip(*this, o, [](auto x, auto y) { return x * y; });
}
template <class U>
MatX<U> cast() const {
    return internal::map1(*this, [](const Scalar& x) { return U(x); });
}
template <class O>
Scalar dot(const O& o) const {
    const auto a = cview();
    const auto b = o.cview();
    if (a.size() != b.size()) throw std::invalid_argument("Eigen shim: dot of vectors of different sizes");
    Scalar acc(0);
    for (Index i = 0; i < a.size(); ++i) acc += internal::cj(a.coeff(i)) * Scalar(b.coeff(i));
    return acc;
}
template <class O>
MatX<Scalar> cross(const O& o) const {
    const auto a = cview();
    const auto b = o.cview();
    if (a.size() != 3 || b.size() != 3) throw std::invalid_argument("Eigen shim: cross needs 3-vectors");
    MatX<Scalar> r(3, 1);
    r(0, 0) = a.coeff(1) * b.coeff(2) - a.coeff(2) * b.coeff(1);
    r(1, 0) = a.coeff(2) * b.coeff(0) - a.coeff(0) * b.coeff(2);
    r(2, 0) = a.coeff(0) * b.coeff(1) - a.coeff(1) * b.coeff(0);
    return r;
}
MatX<Scalar> normalized() const {
    const RealScalar n = norm();
    return internal::map1(*this, [n](const Scalar& x) { return n > 0 ? Scalar(x / n) : x; });
}
// extreme coefficients (real scalars only, as in Eigen)
RealScalar maxCoeff() const {
    Index i = 0, j = 0;
    return ext(&i, &j, true);
}
RealScalar minCoeff() const {
    Index i = 0, j = 0;
    return ext(&i, &j, false);
}
RealScalar maxCoeff(Index* r, Index* c) const { return ext(r, c, true); }
RealScalar minCoeff(Index* r, Index* c) const { return ext(r, c, false); }
RealScalar maxCoeff(Index* k) const {
    Index i = 0, j = 0;
    const RealScalar v = ext(&i, &j, true);
    *k = cols() == 1 ? i : (rows() == 1 ? j : i + rows() * j);
    return v;
}
RealScalar minCoeff(Index* k) const {
    Index i = 0, j = 0;
    const RealScalar v = ext(&i, &j, false);
    *k = cols() == 1 ? i : (rows() == 1 ? j : i + rows() * j);
    return v;
}
RealScalar ext(Index* r, Index* c, bool mx) const {
    static_assert(!internal::is_complex<Scalar>::value, "maxCoeff / minCoeff need real coefficients");
    const auto s = cview();
    if (s.size() == 0) throw std::invalid_argument("Eigen shim: extreme coefficient of an empty matrix");
    RealScalar best = s.coeff(0, 0);
    *r = 0;
    *c = 0;
    for (Index j = 0; j < s.cols(); ++j)
        for (Index i = 0; i < s.rows(); ++i) {
            const RealScalar v = s.coeff(i, j);
            if (mx ? v > best : v < best) {
                best = v;
                *r = i;
                *c = j;
            }
        }
    return best;
}
bool allFinite() const {
    const auto s = cview();
    for (Index j = 0; j < s.cols(); ++j)
        for (Index i = 0; i < s.rows(); ++i)
            if (!std::isfinite(std::abs(s.coeff(i, j)))) return false;
    return true;
}
