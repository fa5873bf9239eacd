// eigen_subset.hpp — TEST INFRASTRUCTURE ONLY (oracle/_ref build).
//
// A clean-room header implementing the subset of the Eigen 3 API that the
// reference's sources and tests use (SURVEY.md §8(c) "Recommended oracle"),
// so /root/reference/proj/src/*.cpp and tests/*.cpp compile in place,
// unmodified, into oracle/_ref. Eigen itself is not in this image and is not
// vendored by the reference (proj/CMakeLists.txt:14).
//
// Evaluation is eager (no expression templates). Rounding order, stated
// because Eigen does not pin it (it depends on version and SIMD width):
//   * products:   r(i,j) = ((a(i,0)*b(0,j) + a(i,1)*b(1,j)) + ...) — k ascending
//   * reductions: sum / squaredNorm / dot / trace run left to right over the
//                 column-major linear index
//   * determinant: Eigen's cofactor expansion along the first row
//   * diagonal products scale rows / columns (no zero terms are added)
// JacobiSVD<3x3> is the two-sided Jacobi sweep (real_2x2_jacobi_svd +
// makeJacobi), descending singular values; JacobiSVD<Dynamic> (test-only) is
// one-sided Jacobi. SelfAdjointEigenSolver<3x3> is cyclic Jacobi, ascending.
// umeyama follows Umeyama (1991) as Eigen documents it.
#pragma once

#include <algorithm>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <initializer_list>
#include <limits>
#include <stdexcept>
#include <type_traits>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;

enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
enum DecompositionOptions {
  ComputeFullU = 0x04,
  ComputeThinU = 0x08,
  ComputeFullV = 0x10,
  ComputeThinV = 0x20,
};

template <typename T, int R, int C>
class Matrix;
template <typename T, int R, int C>
class Array;
template <typename T, int R, int C>
class Block;
template <typename T, int R, int C>
class ArrayRef;
template <typename T, int N>
class DiagonalMatrix;

namespace detail {

inline void size_check(bool ok, const char* what) {
  if (!ok) throw std::logic_error(std::string("eigen_subset: size mismatch in ") + what);
}

template <typename T, int R, int C, bool Fixed = (R != Dynamic && C != Dynamic)>
struct Storage;

template <typename T, int R, int C>
struct Storage<T, R, C, true> {
  T d[R * C];
  constexpr Index rows() const { return R; }
  constexpr Index cols() const { return C; }
  T* ptr() { return d; }
  const T* ptr() const { return d; }
  void resize(Index r, Index c) { size_check(r == R && c == C, "resize"); }
};

template <typename T, int R, int C>
struct Storage<T, R, C, false> {
  std::vector<T> d;
  Index r_ = (R == Dynamic ? 0 : R);
  Index c_ = (C == Dynamic ? 0 : C);
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  T* ptr() { return d.data(); }
  const T* ptr() const { return d.data(); }
  void resize(Index r, Index c) {
    size_check((R == Dynamic || r == R) && (C == Dynamic || c == C), "resize");
    r_ = r;
    c_ = c;
    d.assign(static_cast<std::size_t>(r * c), T(0));
  }
};

constexpr int prod_dim(int a, int b) { return (a == Dynamic || b == Dynamic) ? Dynamic : a; }

}  // namespace detail

// Comma initializer: fills row by row (Eigen's order).
template <typename M>
class CommaInit {
 public:
  CommaInit(M& m, typename M::Scalar first) : m_(m) { put(first); }
  CommaInit& operator,(typename M::Scalar v) {
    put(v);
    return *this;
  }

 private:
  void put(typename M::Scalar v) {
    Index r = k_ / m_.cols(), c = k_ % m_.cols();
    detail::size_check(r < m_.rows(), "comma initializer");
    m_(r, c) = v;
    ++k_;
  }
  M& m_;
  Index k_ = 0;
};

template <typename T, int R, int C>
class Matrix : public detail::Storage<T, R, C> {
  using Base = detail::Storage<T, R, C>;

 public:
  using Scalar = T;
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;
  static constexpr bool IsFixed = (R != Dynamic && C != Dynamic);

  Matrix() {
    if constexpr (IsFixed) {
      for (int k = 0; k < R * C; ++k) this->d[k] = T(0);
    }
  }
  // Vector coefficients (fixed size) or (rows, cols) (dynamic).
  template <typename A, typename B,
            typename = std::enable_if_t<std::is_arithmetic_v<A> && std::is_arithmetic_v<B>>>
  Matrix(A a, B b) {
    if constexpr (IsFixed) {
      static_assert(R * C == 2, "two-coefficient constructor");
      this->d[0] = T(a);
      this->d[1] = T(b);
    } else {
      if constexpr (R == Dynamic && C == Dynamic) {
        Base::resize(Index(a), Index(b));
      } else {
        Base::resize(R == Dynamic ? Index(a) : R, C == Dynamic ? Index(b) : C);
      }
    }
  }
  template <typename A, typename = std::enable_if_t<std::is_integral_v<A>>>
  explicit Matrix(A n) {
    static_assert(!IsFixed, "size constructor on a fixed matrix");
    if constexpr (C == 1) Base::resize(Index(n), 1);
    else Base::resize(1, Index(n));
  }
  Matrix(T a, T b, T c) {
    static_assert(R * C == 3, "three-coefficient constructor");
    this->d[0] = a;
    this->d[1] = b;
    this->d[2] = c;
  }
  Matrix(T a, T b, T c, T e) {
    static_assert(R * C == 4, "four-coefficient constructor");
    this->d[0] = a;
    this->d[1] = b;
    this->d[2] = c;
    this->d[3] = e;
  }
  Matrix(const Block<T, R, C>& b) : Matrix(b.eval()) {}
  Matrix(const Array<T, R, C>& a) : Matrix(a.matrix()) {}
  Matrix(const ArrayRef<T, R, C>& a) : Matrix(a.matrix()) {}
  Matrix(const DiagonalMatrix<T, R>& dm) : Matrix(dm.toDenseMatrix()) {}
  // Fixed <-> dynamic conversions (size checked at run time).
  template <int R2, int C2,
            typename = std::enable_if_t<(R2 != R || C2 != C) && (R2 == R || R2 == Dynamic || R == Dynamic) &&
                                        (C2 == C || C2 == Dynamic || C == Dynamic)>>
  Matrix(const Matrix<T, R2, C2>& o) {
    resize(o.rows(), o.cols());
    for (Index k = 0; k < o.size(); ++k) this->ptr()[k] = o.ptr()[k];
  }

  using Base::cols;
  using Base::rows;
  Index size() const { return rows() * cols(); }
  void resize(Index r, Index c) { Base::resize(r, c); }
  void resize(Index n) {
    if constexpr (C == 1) Base::resize(n, 1);
    else Base::resize(1, n);
  }

  T* data() { return this->ptr(); }
  const T* data() const { return this->ptr(); }

  T& operator()(Index i, Index j) { return this->ptr()[i + j * rows()]; }
  const T& operator()(Index i, Index j) const { return this->ptr()[i + j * rows()]; }
  T& operator()(Index k) { return this->ptr()[k]; }
  const T& operator()(Index k) const { return this->ptr()[k]; }
  T& operator[](Index k) { return this->ptr()[k]; }
  const T& operator[](Index k) const { return this->ptr()[k]; }
  T& coeffRef(Index k) { return this->ptr()[k]; }
  T coeff(Index i, Index j) const { return (*this)(i, j); }

  T& x() { return (*this)(0); }
  T& y() { return (*this)(1); }
  T& z() { return (*this)(2); }
  T& w() { return (*this)(3); }
  T x() const { return (*this)(0); }
  T y() const { return (*this)(1); }
  T z() const { return (*this)(2); }
  T w() const { return (*this)(3); }

  CommaInit<Matrix> operator<<(T v) { return CommaInit<Matrix>(*this, v); }

  static Matrix Zero() {
    static_assert(IsFixed, "Zero() needs sizes");
    return Matrix();
  }
  static Matrix Zero(Index r, Index c) {
    Matrix m;
    m.resize(r, c);
    for (Index k = 0; k < m.size(); ++k) m.ptr()[k] = T(0);
    return m;
  }
  static Matrix Zero(Index n) {
    Matrix m;
    m.resize(n);
    return m;
  }
  static Matrix Constant(T v) {
    static_assert(IsFixed, "Constant() needs sizes");
    Matrix m;
    for (int k = 0; k < R * C; ++k) m.d[k] = v;
    return m;
  }
  static Matrix Ones() { return Constant(T(1)); }
  static Matrix Identity() {
    static_assert(IsFixed, "Identity() needs sizes");
    Matrix m;
    for (int k = 0; k < std::min(R, C); ++k) m(k, k) = T(1);
    return m;
  }
  static Matrix Identity(Index r, Index c) {
    Matrix m = Zero(r, c);
    for (Index k = 0; k < std::min(r, c); ++k) m(k, k) = T(1);
    return m;
  }
  static Matrix Unit(Index i) {
    Matrix m;
    m(i) = T(1);
    return m;
  }
  static Matrix UnitX() { return Unit(0); }
  static Matrix UnitY() { return Unit(1); }
  static Matrix UnitZ() { return Unit(2); }

  Matrix& setZero() {
    for (Index k = 0; k < size(); ++k) this->ptr()[k] = T(0);
    return *this;
  }
  Matrix& setIdentity() {
    setZero();
    for (Index k = 0; k < std::min(rows(), cols()); ++k) (*this)(k, k) = T(1);
    return *this;
  }
  Matrix& setConstant(T v) {
    for (Index k = 0; k < size(); ++k) this->ptr()[k] = v;
    return *this;
  }
  const Matrix& eval() const { return *this; }

  // ---- element-wise arithmetic (hidden friends: found by ADL, allow conversions)
  friend Matrix operator+(const Matrix& a, const Matrix& b) {
    detail::size_check(a.rows() == b.rows() && a.cols() == b.cols(), "+");
    Matrix r = a;
    for (Index k = 0; k < r.size(); ++k) r.ptr()[k] = a.ptr()[k] + b.ptr()[k];
    return r;
  }
  friend Matrix operator-(const Matrix& a, const Matrix& b) {
    detail::size_check(a.rows() == b.rows() && a.cols() == b.cols(), "-");
    Matrix r = a;
    for (Index k = 0; k < r.size(); ++k) r.ptr()[k] = a.ptr()[k] - b.ptr()[k];
    return r;
  }
  friend Matrix operator-(const Matrix& a) {
    Matrix r = a;
    for (Index k = 0; k < r.size(); ++k) r.ptr()[k] = -a.ptr()[k];
    return r;
  }
  friend Matrix operator*(const Matrix& a, T s) {
    Matrix r = a;
    for (Index k = 0; k < r.size(); ++k) r.ptr()[k] = a.ptr()[k] * s;
    return r;
  }
  friend Matrix operator*(T s, const Matrix& a) {
    Matrix r = a;
    for (Index k = 0; k < r.size(); ++k) r.ptr()[k] = s * a.ptr()[k];
    return r;
  }
  friend Matrix operator/(const Matrix& a, T s) {
    Matrix r = a;
    for (Index k = 0; k < r.size(); ++k) r.ptr()[k] = a.ptr()[k] / s;
    return r;
  }
  friend bool operator==(const Matrix& a, const Matrix& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
    for (Index k = 0; k < a.size(); ++k)
      if (!(a.ptr()[k] == b.ptr()[k])) return false;
    return true;
  }
  friend bool operator!=(const Matrix& a, const Matrix& b) { return !(a == b); }

  Matrix& operator+=(const Matrix& b) { return *this = *this + b; }
  Matrix& operator-=(const Matrix& b) { return *this = *this - b; }
  Matrix& operator*=(T s) { return *this = *this * s; }
  Matrix& operator/=(T s) { return *this = *this / s; }
  Matrix& operator*=(const Matrix& b) { return *this = (*this) * b; }

  // ---- products
  template <int R2, int C2>
  Matrix<T, R, C2> operator*(const Matrix<T, R2, C2>& b) const {
    static_assert(C == R2 || C == Dynamic || R2 == Dynamic, "inner dimensions");
    detail::size_check(cols() == b.rows(), "product");
    Matrix<T, R, C2> r;
    r.resize(rows(), b.cols());
    for (Index i = 0; i < rows(); ++i)
      for (Index j = 0; j < b.cols(); ++j) {
        T acc = (*this)(i, 0) * b(0, j);
        for (Index k = 1; k < cols(); ++k) acc = acc + (*this)(i, k) * b(k, j);
        r(i, j) = acc;
      }
    return r;
  }
  Matrix operator*(const DiagonalMatrix<T, C>& dm) const {  // column scaling
    Matrix r = *this;
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) r(i, j) = (*this)(i, j) * dm.diagonal()(j);
    return r;
  }

  // ---- reductions and norms (left to right over the storage order)
  T sum() const {
    T acc = this->ptr()[0];
    for (Index k = 1; k < size(); ++k) acc = acc + this->ptr()[k];
    return acc;
  }
  T mean() const { return sum() / T(size()); }
  T squaredNorm() const {
    T acc = this->ptr()[0] * this->ptr()[0];
    for (Index k = 1; k < size(); ++k) acc = acc + this->ptr()[k] * this->ptr()[k];
    return acc;
  }
  T norm() const { return std::sqrt(squaredNorm()); }
  T dot(const Matrix& b) const {
    detail::size_check(size() == b.size(), "dot");
    T acc = this->ptr()[0] * b.ptr()[0];
    for (Index k = 1; k < size(); ++k) acc = acc + this->ptr()[k] * b.ptr()[k];
    return acc;
  }
  T trace() const {
    T acc = (*this)(0, 0);
    for (Index k = 1; k < std::min(rows(), cols()); ++k) acc = acc + (*this)(k, k);
    return acc;
  }
  T maxCoeff() const {
    T m = this->ptr()[0];
    for (Index k = 1; k < size(); ++k) m = std::max(m, this->ptr()[k]);
    return m;
  }
  T minCoeff() const {
    T m = this->ptr()[0];
    for (Index k = 1; k < size(); ++k) m = std::min(m, this->ptr()[k]);
    return m;
  }
  template <typename I>
  T maxCoeff(I* idx) const {
    Index best = 0;
    for (Index k = 1; k < size(); ++k)
      if (this->ptr()[k] > this->ptr()[best]) best = k;
    *idx = static_cast<I>(best);
    return this->ptr()[best];
  }
  Matrix normalized() const {
    T z = squaredNorm();
    if (z > T(0)) return *this / std::sqrt(z);
    return *this;
  }
  void normalize() { *this = normalized(); }
  bool allFinite() const {
    for (Index k = 0; k < size(); ++k)
      if (!std::isfinite(this->ptr()[k])) return false;
    return true;
  }
  bool hasNaN() const {
    for (Index k = 0; k < size(); ++k)
      if (std::isnan(this->ptr()[k])) return true;
    return false;
  }
  bool isZero(T prec = T(1e-12)) const {
    for (Index k = 0; k < size(); ++k)
      if (!(std::abs(this->ptr()[k]) <= prec)) return false;
    return true;
  }
  bool isApprox(const Matrix& o, T prec = T(1e-12)) const {
    return (*this - o).squaredNorm() <= prec * prec * std::min(squaredNorm(), o.squaredNorm());
  }

  Matrix cwiseAbs() const {
    Matrix r = *this;
    for (Index k = 0; k < size(); ++k) r.ptr()[k] = std::abs(this->ptr()[k]);
    return r;
  }
  Matrix cwiseProduct(const Matrix& b) const {
    Matrix r = *this;
    for (Index k = 0; k < size(); ++k) r.ptr()[k] = this->ptr()[k] * b.ptr()[k];
    return r;
  }
  Matrix cwiseQuotient(const Matrix& b) const {
    Matrix r = *this;
    for (Index k = 0; k < size(); ++k) r.ptr()[k] = this->ptr()[k] / b.ptr()[k];
    return r;
  }
  Matrix cwiseMin(const Matrix& b) const {
    Matrix r = *this;
    for (Index k = 0; k < size(); ++k) r.ptr()[k] = std::min(this->ptr()[k], b.ptr()[k]);
    return r;
  }
  Matrix cwiseMax(const Matrix& b) const {
    Matrix r = *this;
    for (Index k = 0; k < size(); ++k) r.ptr()[k] = std::max(this->ptr()[k], b.ptr()[k]);
    return r;
  }
  Matrix cwiseMin(T s) const { return cwiseMin(Matrix(*this).setConstant(s)); }
  Matrix cwiseMax(T s) const { return cwiseMax(Matrix(*this).setConstant(s)); }

  Matrix<T, C, R> transpose() const {
    Matrix<T, C, R> r;
    r.resize(cols(), rows());
    for (Index i = 0; i < rows(); ++i)
      for (Index j = 0; j < cols(); ++j) r(j, i) = (*this)(i, j);
    return r;
  }

  Matrix<T, 3, 1> cross(const Matrix<T, 3, 1>& b) const {
    static_assert(R == 3 && C == 1, "cross of 3-vectors");
    const Matrix& a = *this;
    return Matrix<T, 3, 1>(a(1) * b(2) - a(2) * b(1), a(2) * b(0) - a(0) * b(2), a(0) * b(1) - a(1) * b(0));
  }

  T determinant() const {
    detail::size_check(rows() == cols(), "determinant");
    const Matrix& m = *this;
    if (rows() == 1) return m(0, 0);
    if (rows() == 2) return m(0, 0) * m(1, 1) - m(1, 0) * m(0, 1);
    if (rows() == 3) {
      // bruteforce_det3_helper(m,0,1,2) - (m,1,0,2) + (m,2,0,1) in Eigen's layout.
      auto h = [&](int a, int b, int c) { return m(0, a) * (m(1, b) * m(2, c) - m(1, c) * m(2, b)); };
      return h(0, 1, 2) - h(1, 0, 2) + h(2, 0, 1);
    }
    // Partial-pivot LU for larger sizes (not on the reference's hot path).
    Matrix a = m;
    T det = T(1);
    const Index n = rows();
    for (Index k = 0; k < n; ++k) {
      Index p = k;
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(a(i, k)) > std::abs(a(p, k))) p = i;
      if (a(p, k) == T(0)) return T(0);
      if (p != k) {
        for (Index j = 0; j < n; ++j) std::swap(a(k, j), a(p, j));
        det = -det;
      }
      det *= a(k, k);
      for (Index i = k + 1; i < n; ++i) {
        T f = a(i, k) / a(k, k);
        for (Index j = k; j < n; ++j) a(i, j) -= f * a(k, j);
      }
    }
    return det;
  }

  Matrix inverse() const {
    detail::size_check(rows() == cols(), "inverse");
    const Matrix& m = *this;
    Matrix r = m;
    if (rows() == 2) {
      T det = m.determinant();
      r(0, 0) = m(1, 1) / det;
      r(1, 1) = m(0, 0) / det;
      r(0, 1) = -m(0, 1) / det;
      r(1, 0) = -m(1, 0) / det;
      return r;
    }
    if (rows() == 3) {
      auto cof = [&](int i, int j) {
        int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
        return m(i1, j1) * m(i2, j2) - m(i1, j2) * m(i2, j1);
      };
      T c00 = cof(0, 0), c10 = cof(1, 0), c20 = cof(2, 0);
      T det = c00 * m(0, 0) + c10 * m(1, 0) + c20 * m(2, 0);
      T inv = T(1) / det;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r(i, j) = cof(j, i) * inv;
      return r;
    }
    // Gauss-Jordan for other sizes.
    const Index n = rows();
    Matrix a = m;
    r.setIdentity();
    for (Index k = 0; k < n; ++k) {
      Index p = k;
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(a(i, k)) > std::abs(a(p, k))) p = i;
      for (Index j = 0; j < n; ++j) {
        std::swap(a(k, j), a(p, j));
        std::swap(r(k, j), r(p, j));
      }
      T piv = a(k, k);
      for (Index j = 0; j < n; ++j) {
        a(k, j) /= piv;
        r(k, j) /= piv;
      }
      for (Index i = 0; i < n; ++i) {
        if (i == k) continue;
        T f = a(i, k);
        for (Index j = 0; j < n; ++j) {
          a(i, j) -= f * a(k, j);
          r(i, j) -= f * r(k, j);
        }
      }
    }
    return r;
  }

  DiagonalMatrix<T, R> asDiagonal() const;

  // ---- blocks (writable views)
  Block<T, 1, C> row(Index i) { return Block<T, 1, C>(&(*this)(i, 0), rows(), 1, cols()); }
  Block<T, R, 1> col(Index j) { return Block<T, R, 1>(&(*this)(0, j), rows(), rows(), 1); }
  Matrix<T, 1, C> row(Index i) const { return Block<T, 1, C>(const_cast<T*>(&(*this)(i, 0)), rows(), 1, cols()).eval(); }
  Matrix<T, R, 1> col(Index j) const { return Block<T, R, 1>(const_cast<T*>(&(*this)(0, j)), rows(), rows(), 1).eval(); }
  template <int N>
  Block<T, N, 1> head() { return Block<T, N, 1>(data(), rows(), N, 1); }
  template <int N>
  Block<T, N, 1> tail() { return Block<T, N, 1>(data() + (size() - N), rows(), N, 1); }
  template <int N>
  Matrix<T, N, 1> head() const { return const_cast<Matrix*>(this)->template head<N>().eval(); }
  template <int N>
  Matrix<T, N, 1> tail() const { return const_cast<Matrix*>(this)->template tail<N>().eval(); }
  template <int BR, int BC>
  Block<T, BR, BC> block(Index i, Index j) { return Block<T, BR, BC>(&(*this)(i, j), rows(), BR, BC); }
  template <int BR, int BC>
  Matrix<T, BR, BC> block(Index i, Index j) const {
    return const_cast<Matrix*>(this)->template block<BR, BC>(i, j).eval();
  }
  template <int BR, int BC>
  Block<T, BR, BC> topLeftCorner() { return block<BR, BC>(0, 0); }
  template <int BR, int BC>
  Block<T, BR, BC> topRightCorner() { return block<BR, BC>(0, cols() - BC); }
  template <int BR, int BC>
  Block<T, BR, BC> bottomLeftCorner() { return block<BR, BC>(rows() - BR, 0); }
  template <int BR, int BC>
  Block<T, BR, BC> bottomRightCorner() { return block<BR, BC>(rows() - BR, cols() - BC); }
  template <int BR, int BC>
  Matrix<T, BR, BC> topLeftCorner() const { return block<BR, BC>(0, 0); }
  template <int BR, int BC>
  Matrix<T, BR, BC> topRightCorner() const { return block<BR, BC>(0, cols() - BC); }
  template <int BR, int BC>
  Matrix<T, BR, BC> bottomLeftCorner() const { return block<BR, BC>(rows() - BR, 0); }
  template <int BR, int BC>
  Matrix<T, BR, BC> bottomRightCorner() const { return block<BR, BC>(rows() - BR, cols() - BC); }
  template <int N>
  Block<T, R, N> leftCols() { return Block<T, R, N>(data(), rows(), rows(), N); }
  template <int N>
  Block<T, R, N> rightCols() { return Block<T, R, N>(&(*this)(0, cols() - N), rows(), rows(), N); }
  template <int N>
  Matrix<T, R, N> leftCols() const { return const_cast<Matrix*>(this)->template leftCols<N>().eval(); }
  template <int N>
  Matrix<T, R, N> rightCols() const { return const_cast<Matrix*>(this)->template rightCols<N>().eval(); }

  // ---- array view
  ArrayRef<T, R, C> array() { return ArrayRef<T, R, C>(this); }
  Array<T, R, C> array() const;

  // ---- partial reductions (rowwise().mean(), colwise() - v)
  struct Rowwise {
    const Matrix* m;
    Matrix<T, R, 1> sum() const {
      Matrix<T, R, 1> r;
      r.resize(m->rows(), 1);
      for (Index i = 0; i < m->rows(); ++i) {
        T acc = (*m)(i, 0);
        for (Index j = 1; j < m->cols(); ++j) acc = acc + (*m)(i, j);
        r(i) = acc;
      }
      return r;
    }
    Matrix<T, R, 1> mean() const { return sum() / T(m->cols()); }
    Matrix<T, R, 1> squaredNorm() const {
      Matrix<T, R, 1> r;
      r.resize(m->rows(), 1);
      for (Index i = 0; i < m->rows(); ++i) {
        T acc = (*m)(i, 0) * (*m)(i, 0);
        for (Index j = 1; j < m->cols(); ++j) acc = acc + (*m)(i, j) * (*m)(i, j);
        r(i) = acc;
      }
      return r;
    }
  };
  struct Colwise {
    const Matrix* m;
    template <int VR>
    friend Matrix operator-(const Colwise& cw, const Matrix<T, VR, 1>& v) {
      detail::size_check(v.rows() == cw.m->rows(), "colwise -");
      Matrix r = *cw.m;
      for (Index j = 0; j < r.cols(); ++j)
        for (Index i = 0; i < r.rows(); ++i) r(i, j) = (*cw.m)(i, j) - v(i);
      return r;
    }
    template <int VR>
    friend Matrix operator+(const Colwise& cw, const Matrix<T, VR, 1>& v) {
      Matrix r = *cw.m;
      for (Index j = 0; j < r.cols(); ++j)
        for (Index i = 0; i < r.rows(); ++i) r(i, j) = (*cw.m)(i, j) + v(i);
      return r;
    }
    Matrix<T, 1, C> sum() const {
      Matrix<T, 1, C> r;
      r.resize(1, m->cols());
      for (Index j = 0; j < m->cols(); ++j) {
        T acc = (*m)(0, j);
        for (Index i = 1; i < m->rows(); ++i) acc = acc + (*m)(i, j);
        r(j) = acc;
      }
      return r;
    }
    Matrix<T, 1, C> mean() const { return sum() / T(m->rows()); }
  };
  Rowwise rowwise() const { return Rowwise{this}; }
  Colwise colwise() const { return Colwise{this}; }
};

// ---------------------------------------------------------------- Block view
template <typename T, int BR, int BC>
class Block {
 public:
  using Scalar = T;
  using Mat = Matrix<T, BR, BC>;
  Block(T* p, Index ld, Index r, Index c) : p_(p), ld_(ld), r_(r), c_(c) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  T& operator()(Index i, Index j) const { return p_[i + j * ld_]; }
  T& operator()(Index k) const { return r_ == 1 ? p_[k * ld_] : p_[k]; }

  Mat eval() const {
    Mat m;
    m.resize(r_, c_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) m(i, j) = (*this)(i, j);
    return m;
  }

  Block& operator=(const Block& o) { return assign(o.eval()); }
  template <int R2, int C2>
  Block& operator=(const Matrix<T, R2, C2>& m) {
    return assign(m);
  }
  Block& operator*=(T s) {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*this)(i, j) *= s;
    return *this;
  }
  Block& operator/=(T s) {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*this)(i, j) /= s;
    return *this;
  }
  Block& operator+=(const Mat& m) { return assign(eval() + m); }
  Block& operator-=(const Mat& m) { return assign(eval() - m); }

  T norm() const { return eval().norm(); }
  T squaredNorm() const { return eval().squaredNorm(); }
  T sum() const { return eval().sum(); }
  T dot(const Mat& b) const { return eval().dot(b); }
  Matrix<T, BC, BR> transpose() const { return eval().transpose(); }
  Mat normalized() const { return eval().normalized(); }
  Mat cwiseAbs() const { return eval().cwiseAbs(); }
  T maxCoeff() const { return eval().maxCoeff(); }
  bool allFinite() const { return eval().allFinite(); }
  Matrix<T, 3, 1> cross(const Matrix<T, 3, 1>& b) const { return eval().cross(b); }
  T x() const { return (*this)(0); }
  T y() const { return (*this)(1); }
  T z() const { return (*this)(2); }

  friend Mat operator+(const Block& a, const Mat& b) { return a.eval() + b; }
  friend Mat operator+(const Mat& a, const Block& b) { return a + b.eval(); }
  friend Mat operator+(const Block& a, const Block& b) { return a.eval() + b.eval(); }
  friend Mat operator-(const Block& a, const Mat& b) { return a.eval() - b; }
  friend Mat operator-(const Mat& a, const Block& b) { return a - b.eval(); }
  friend Mat operator-(const Block& a, const Block& b) { return a.eval() - b.eval(); }
  friend Mat operator-(const Block& a) { return -a.eval(); }
  friend Mat operator*(T s, const Block& b) { return s * b.eval(); }
  friend Mat operator*(const Block& b, T s) { return b.eval() * s; }
  friend Mat operator/(const Block& b, T s) { return b.eval() / s; }
  template <int R2>
  friend Matrix<T, R2, BC> operator*(const Matrix<T, R2, BR>& a, const Block& b) {
    return a * b.eval();
  }
  template <int C2>
  friend Matrix<T, BR, C2> operator*(const Block& a, const Matrix<T, BC, C2>& b) {
    return a.eval() * b;
  }

 private:
  template <int R2, int C2>
  Block& assign(const Matrix<T, R2, C2>& m) {
    detail::size_check(m.rows() == r_ && m.cols() == c_, "block assignment");
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*this)(i, j) = m(i, j);
    return *this;
  }
  T* p_;
  Index ld_, r_, c_;
};

// ---------------------------------------------------------------- Diagonal
template <typename T, int N>
class DiagonalMatrix {
 public:
  explicit DiagonalMatrix(const Matrix<T, N, 1>& d) : d_(d) {}
  const Matrix<T, N, 1>& diagonal() const { return d_; }
  Matrix<T, N, N> toDenseMatrix() const {
    Matrix<T, N, N> m = Matrix<T, N, N>::Zero(d_.size(), d_.size());
    for (Index k = 0; k < d_.size(); ++k) m(k, k) = d_(k);
    return m;
  }
  template <int C2>
  friend Matrix<T, N, C2> operator*(const DiagonalMatrix& dm, const Matrix<T, N, C2>& b) {  // row scaling
    Matrix<T, N, C2> r = b;
    for (Index j = 0; j < b.cols(); ++j)
      for (Index i = 0; i < b.rows(); ++i) r(i, j) = dm.d_(i) * b(i, j);
    return r;
  }

 private:
  Matrix<T, N, 1> d_;
};

template <typename T, int R, int C>
DiagonalMatrix<T, R> Matrix<T, R, C>::asDiagonal() const {
  static_assert(C == 1, "asDiagonal of a column vector");
  return DiagonalMatrix<T, R>(*this);
}

// ---------------------------------------------------------------- Array
template <typename T, int R, int C>
class Array {
 public:
  using Scalar = T;
  Array() = default;
  explicit Array(const Matrix<T, R, C>& m) : m_(m) {}
  const Matrix<T, R, C>& matrix() const { return m_; }
  Index size() const { return m_.size(); }
  T operator()(Index k) const { return m_(k); }

  template <typename F>
  Array map(F f) const {
    Array r(m_);
    for (Index k = 0; k < size(); ++k) r.m_.data()[k] = f(m_.data()[k]);
    return r;
  }
  Array exp() const { return map([](T v) { return std::exp(v); }); }
  Array log() const { return map([](T v) { return std::log(v); }); }
  Array sqrt() const { return map([](T v) { return std::sqrt(v); }); }
  Array abs() const { return map([](T v) { return std::abs(v); }); }
  Array square() const { return map([](T v) { return v * v; }); }
  Array inverse() const { return map([](T v) { return T(1) / v; }); }
  T sum() const { return m_.sum(); }
  T maxCoeff() const { return m_.maxCoeff(); }
  T minCoeff() const { return m_.minCoeff(); }

  friend Array operator*(const Array& a, const Array& b) { return Array(a.m_.cwiseProduct(b.m_)); }
  friend Array operator/(const Array& a, const Array& b) { return Array(a.m_.cwiseQuotient(b.m_)); }
  friend Array operator+(const Array& a, const Array& b) { return Array(a.m_ + b.m_); }
  friend Array operator-(const Array& a, const Array& b) { return Array(a.m_ - b.m_); }
  friend Array operator*(const Array& a, T s) { return Array(a.m_ * s); }
  friend Array operator*(T s, const Array& a) { return Array(s * a.m_); }
  friend Array operator/(const Array& a, T s) { return Array(a.m_ / s); }
  friend Array operator+(const Array& a, T s) { return a.map([s](T v) { return v + s; }); }
  friend Array operator-(const Array& a, T s) { return a.map([s](T v) { return v - s; }); }
  friend Array operator+(T s, const Array& a) { return a.map([s](T v) { return s + v; }); }
  friend Array operator-(T s, const Array& a) { return a.map([s](T v) { return s - v; }); }

 private:
  Matrix<T, R, C> m_;
};

template <typename T, int R, int C>
Array<T, R, C> Matrix<T, R, C>::array() const {
  return Array<T, R, C>(*this);
}

// Writable array view of a matrix (l.array() += s).
template <typename T, int R, int C>
class ArrayRef {
 public:
  explicit ArrayRef(Matrix<T, R, C>* m) : m_(m) {}
  Array<T, R, C> val() const { return Array<T, R, C>(*m_); }
  operator Array<T, R, C>() const { return val(); }
  const Matrix<T, R, C>& matrix() const { return *m_; }
  Array<T, R, C> exp() const { return val().exp(); }
  Array<T, R, C> log() const { return val().log(); }
  Array<T, R, C> sqrt() const { return val().sqrt(); }
  Array<T, R, C> abs() const { return val().abs(); }
  Array<T, R, C> square() const { return val().square(); }
  T sum() const { return m_->sum(); }
  T maxCoeff() const { return m_->maxCoeff(); }
  ArrayRef& operator+=(T s) {
    for (Index k = 0; k < m_->size(); ++k) m_->data()[k] += s;
    return *this;
  }
  ArrayRef& operator-=(T s) {
    for (Index k = 0; k < m_->size(); ++k) m_->data()[k] -= s;
    return *this;
  }
  ArrayRef& operator*=(T s) {
    for (Index k = 0; k < m_->size(); ++k) m_->data()[k] *= s;
    return *this;
  }
  ArrayRef& operator*=(const Array<T, R, C>& a) {
    for (Index k = 0; k < m_->size(); ++k) m_->data()[k] *= a(k);
    return *this;
  }
  ArrayRef& operator=(const Array<T, R, C>& a) {
    *m_ = a.matrix();
    return *this;
  }
  friend Array<T, R, C> operator*(const ArrayRef& a, const ArrayRef& b) { return a.val() * b.val(); }
  friend Array<T, R, C> operator*(const ArrayRef& a, const Array<T, R, C>& b) { return a.val() * b; }
  friend Array<T, R, C> operator*(const Array<T, R, C>& a, const ArrayRef& b) { return a * b.val(); }
  friend Array<T, R, C> operator/(const ArrayRef& a, const ArrayRef& b) { return a.val() / b.val(); }
  friend Array<T, R, C> operator+(const ArrayRef& a, const ArrayRef& b) { return a.val() + b.val(); }
  friend Array<T, R, C> operator-(const ArrayRef& a, const ArrayRef& b) { return a.val() - b.val(); }
  friend Array<T, R, C> operator*(const ArrayRef& a, T s) { return a.val() * s; }
  friend Array<T, R, C> operator*(T s, const ArrayRef& a) { return s * a.val(); }
  friend Array<T, R, C> operator/(const ArrayRef& a, T s) { return a.val() / s; }
  friend Array<T, R, C> operator+(const ArrayRef& a, T s) { return a.val() + s; }
  friend Array<T, R, C> operator-(const ArrayRef& a, T s) { return a.val() - s; }
  friend Array<T, R, C> operator-(T s, const ArrayRef& a) { return s - a.val(); }

 private:
  Matrix<T, R, C>* m_;
};

}  // namespace Eigen
