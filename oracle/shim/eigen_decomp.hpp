// eigen_decomp.hpp — TEST INFRASTRUCTURE ONLY (oracle/_ref build).
//
// Clean-room decompositions for the Eigen-subset shim (see eigen_subset.hpp):
// JacobiSVD, SelfAdjointEigenSolver, LLT, Quaternion-from-rotation and
// umeyama, restated from the published algorithms Eigen documents.
#pragma once

#include "eigen_subset.hpp"

#include <utility>

namespace Eigen {

namespace detail {

struct JRot {
  double c, s;
};

// JacobiRotation::applyOnTheLeft(p, q, j): rows p, q.
template <typename M>
void rot_rows(M& m, Index p, Index q, JRot j) {
  for (Index i = 0; i < m.cols(); ++i) {
    double x = m(p, i), y = m(q, i);
    m(p, i) = j.c * x + j.s * y;
    m(q, i) = -j.s * x + j.c * y;
  }
}
// JacobiRotation::applyOnTheRight(p, q, j): columns p, q with j^T.
template <typename M>
void rot_cols(M& m, Index p, Index q, JRot j) {
  JRot t{j.c, -j.s};
  for (Index i = 0; i < m.rows(); ++i) {
    double x = m(i, p), y = m(i, q);
    m(i, p) = t.c * x + t.s * y;
    m(i, q) = -t.s * x + t.c * y;
  }
}

// Two-sided Jacobi SVD of a square matrix (real_2x2_jacobi_svd + makeJacobi
// per off-diagonal pair, sweeps until below 2*eps*max|diag|), then sign fix
// and a descending selection sort of the singular values.
template <int N>
void jacobi_svd_square(const Matrix<double, N, N>& a, Matrix<double, N, N>* u_out, Matrix<double, N, 1>* s_out,
                       Matrix<double, N, N>* v_out) {
  const double min_pos = std::numeric_limits<double>::min();
  const double precision = 2.0 * std::numeric_limits<double>::epsilon();
  const Index n = a.rows();
  double scale = a.cwiseAbs().maxCoeff();
  if (scale == 0.0) scale = 1.0;
  Matrix<double, N, N> m = a / scale;
  Matrix<double, N, N> u = Matrix<double, N, N>::Identity(n, n);
  Matrix<double, N, N> v = Matrix<double, N, N>::Identity(n, n);
  double max_diag = 0.0;
  for (Index k = 0; k < n; ++k) max_diag = std::max(max_diag, std::abs(m(k, k)));
  bool finished = false;
  while (!finished) {
    finished = true;
    for (Index p = 1; p < n; ++p) {
      for (Index q = 0; q < p; ++q) {
        double threshold = std::max(min_pos, precision * max_diag);
        if (std::abs(m(p, q)) > threshold || std::abs(m(q, p)) > threshold) {
          finished = false;
          double m00 = m(p, p), m01 = m(p, q), m10 = m(q, p), m11 = m(q, q);
          JRot rot1;
          double t = m00 + m11, d = m10 - m01;
          if (std::abs(d) < min_pos) {
            rot1 = {1.0, 0.0};
          } else {
            double uu = t / d;
            double tmp = std::sqrt(1.0 + uu * uu);
            rot1 = {uu / tmp, 1.0 / tmp};
          }
          double n00 = rot1.c * m00 + rot1.s * m10, n01 = rot1.c * m01 + rot1.s * m11;
          double n11 = -rot1.s * m01 + rot1.c * m11;
          JRot jr;
          double deno = 2.0 * std::abs(n01);
          if (deno < min_pos) {
            jr = {1.0, 0.0};
          } else {
            double tau = (n00 - n11) / deno;
            double w = std::sqrt(tau * tau + 1.0);
            double tt = tau > 0.0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
            double sign_t = tt > 0.0 ? 1.0 : -1.0;
            double nn = 1.0 / std::sqrt(tt * tt + 1.0);
            jr = {nn, -sign_t * (n01 / std::abs(n01)) * std::abs(tt) * nn};
          }
          JRot jrt{jr.c, -jr.s};
          JRot jl{rot1.c * jrt.c - rot1.s * jrt.s, rot1.c * jrt.s + rot1.s * jrt.c};
          rot_rows(m, p, q, jl);
          rot_cols(u, p, q, JRot{jl.c, -jl.s});
          rot_cols(m, p, q, jr);
          rot_cols(v, p, q, jr);
          max_diag = std::max(max_diag, std::max(std::abs(m(p, p)), std::abs(m(q, q))));
        }
      }
    }
  }
  Matrix<double, N, 1> s = Matrix<double, N, 1>::Zero(n);
  for (Index i = 0; i < n; ++i) {
    double d = m(i, i);
    s(i) = std::abs(d);
    if (d < 0.0)
      for (Index r = 0; r < n; ++r) u(r, i) = -u(r, i);
  }
  s = s * scale;
  for (Index i = 0; i < n; ++i) {
    Index best = i;
    for (Index k = i + 1; k < n; ++k)
      if (s(k) > s(best)) best = k;
    if (s(best) == 0.0) break;
    if (best != i) {
      std::swap(s(i), s(best));
      for (Index r = 0; r < n; ++r) {
        std::swap(u(r, i), u(r, best));
        std::swap(v(r, i), v(r, best));
      }
    }
  }
  *u_out = u;
  *s_out = s;
  *v_out = v;
}

}  // namespace detail

template <typename MatrixType>
class JacobiSVD {
 public:
  using T = typename MatrixType::Scalar;
  static constexpr int R = MatrixType::RowsAtCompileTime;
  static constexpr int C = MatrixType::ColsAtCompileTime;

  explicit JacobiSVD(const MatrixType& a, unsigned int = 0) {
    if constexpr (R != Dynamic && R == C) {
      detail::jacobi_svd_square<R>(a, &u_, &s_, &v_);
    } else {
      one_sided(a);
    }
  }
  const Matrix<T, R, R>& matrixU() const { return u_; }
  const Matrix<T, C, C>& matrixV() const { return v_; }
  const Matrix<T, (R == Dynamic || C == Dynamic) ? Dynamic : (R < C ? R : C), 1>& singularValues() const {
    return s_;
  }

 private:
  // One-sided (Hestenes) Jacobi on the columns; singular values only are
  // meaningful for non-square inputs (test-side use: test_scene.cpp:300).
  void one_sided(const MatrixType& a0) {
    Matrix<T, Dynamic, Dynamic> a(a0.rows(), a0.cols());
    for (Index j = 0; j < a0.cols(); ++j)
      for (Index i = 0; i < a0.rows(); ++i) a(i, j) = a0(i, j);
    const Index n = a.cols();
    for (int sweep = 0; sweep < 60; ++sweep) {
      bool rotated = false;
      for (Index p = 0; p < n; ++p)
        for (Index q = p + 1; q < n; ++q) {
          T alpha = 0, beta = 0, gamma = 0;
          for (Index i = 0; i < a.rows(); ++i) {
            alpha += a(i, p) * a(i, p);
            beta += a(i, q) * a(i, q);
            gamma += a(i, p) * a(i, q);
          }
          if (std::abs(gamma) <= 1e-300 || std::abs(gamma) <= 1e-15 * std::sqrt(alpha * beta)) continue;
          rotated = true;
          T zeta = (beta - alpha) / (2 * gamma);
          T t = (zeta >= 0 ? 1 : -1) / (std::abs(zeta) + std::sqrt(1 + zeta * zeta));
          T c = 1 / std::sqrt(1 + t * t), s = c * t;
          for (Index i = 0; i < a.rows(); ++i) {
            T x = a(i, p), y = a(i, q);
            a(i, p) = c * x - s * y;
            a(i, q) = s * x + c * y;
          }
        }
      if (!rotated) break;
    }
    std::vector<T> sv(n);
    for (Index j = 0; j < n; ++j) {
      T acc = 0;
      for (Index i = 0; i < a.rows(); ++i) acc += a(i, j) * a(i, j);
      sv[j] = std::sqrt(acc);
    }
    std::sort(sv.begin(), sv.end(), [](T x, T y) { return x > y; });
    const Index k = std::min(a.rows(), a.cols());
    s_.resize(k);
    for (Index i = 0; i < k; ++i) s_(i) = sv[i];
  }

  Matrix<T, R, R> u_;
  Matrix<T, C, C> v_;
  Matrix<T, (R == Dynamic || C == Dynamic) ? Dynamic : (R < C ? R : C), 1> s_;
};

// Symmetric eigenvalues by cyclic Jacobi rotations, ascending.
template <typename MatrixType>
class SelfAdjointEigenSolver {
 public:
  using T = typename MatrixType::Scalar;
  static constexpr int N = MatrixType::RowsAtCompileTime;
  explicit SelfAdjointEigenSolver(const MatrixType& a0) {
    MatrixType a = a0;
    MatrixType v = MatrixType::Identity();
    const Index n = a.rows();
    for (int sweep = 0; sweep < 100; ++sweep) {
      T off = 0;
      for (Index p = 0; p < n; ++p)
        for (Index q = p + 1; q < n; ++q) off += a(p, q) * a(p, q);
      if (off < 1e-300) break;
      for (Index p = 0; p < n; ++p)
        for (Index q = p + 1; q < n; ++q) {
          if (a(p, q) == 0) continue;
          T theta = (a(q, q) - a(p, p)) / (2 * a(p, q));
          T t = (theta >= 0 ? 1 : -1) / (std::abs(theta) + std::sqrt(theta * theta + 1));
          T c = 1 / std::sqrt(t * t + 1), s = t * c;
          for (Index k = 0; k < n; ++k) {  // A <- J^T A J
            T akp = a(k, p), akq = a(k, q);
            a(k, p) = c * akp - s * akq;
            a(k, q) = s * akp + c * akq;
          }
          for (Index k = 0; k < n; ++k) {
            T apk = a(p, k), aqk = a(q, k);
            a(p, k) = c * apk - s * aqk;
            a(q, k) = s * apk + c * aqk;
          }
          for (Index k = 0; k < n; ++k) {
            T vkp = v(k, p), vkq = v(k, q);
            v(k, p) = c * vkp - s * vkq;
            v(k, q) = s * vkp + c * vkq;
          }
        }
    }
    std::vector<Index> idx(n);
    for (Index k = 0; k < n; ++k) idx[k] = k;
    std::sort(idx.begin(), idx.end(), [&](Index x, Index y) { return a(x, x) < a(y, y); });
    for (Index k = 0; k < n; ++k) {
      evals_(k) = a(idx[k], idx[k]);
      for (Index r = 0; r < n; ++r) evecs_(r, k) = v(r, idx[k]);
    }
  }
  const Matrix<T, N, 1>& eigenvalues() const { return evals_; }
  const MatrixType& eigenvectors() const { return evecs_; }
  ComputationInfo info() const { return Success; }

 private:
  Matrix<T, N, 1> evals_;
  MatrixType evecs_;
};

template <typename MatrixType>
class LLT {
 public:
  using T = typename MatrixType::Scalar;
  explicit LLT(const MatrixType& a) : l_(MatrixType::Zero()) {
    const Index n = a.rows();
    for (Index j = 0; j < n; ++j) {
      T d = a(j, j);
      for (Index k = 0; k < j; ++k) d -= l_(j, k) * l_(j, k);
      if (!(d > 0)) {
        info_ = NumericalIssue;
        return;
      }
      l_(j, j) = std::sqrt(d);
      for (Index i = j + 1; i < n; ++i) {
        T v = a(i, j);
        for (Index k = 0; k < j; ++k) v -= l_(i, k) * l_(j, k);
        l_(i, j) = v / l_(j, j);
      }
    }
  }
  ComputationInfo info() const { return info_; }
  const MatrixType& matrixL() const { return l_; }

 private:
  MatrixType l_;
  ComputationInfo info_ = Success;
};

// Quaternion from a rotation matrix (Shepperd's branch on the trace, as
// Eigen's quaternionbase_assign_impl).
template <typename T>
class Quaternion {
 public:
  Quaternion(T w, T x, T y, T z) : w_(w), x_(x), y_(y), z_(z) {}
  explicit Quaternion(const Matrix<T, 3, 3>& m) {
    T t = m.trace();
    if (t > T(0)) {
      t = std::sqrt(t + T(1));
      w_ = T(0.5) * t;
      t = T(0.5) / t;
      x_ = (m(2, 1) - m(1, 2)) * t;
      y_ = (m(0, 2) - m(2, 0)) * t;
      z_ = (m(1, 0) - m(0, 1)) * t;
    } else {
      int i = 0;
      if (m(1, 1) > m(0, 0)) i = 1;
      if (m(2, 2) > m(i, i)) i = 2;
      int j = (i + 1) % 3, k = (j + 1) % 3;
      t = std::sqrt(m(i, i) - m(j, j) - m(k, k) + T(1));
      T v[3];
      v[i] = T(0.5) * t;
      t = T(0.5) / t;
      w_ = (m(k, j) - m(j, k)) * t;
      v[j] = (m(j, i) + m(i, j)) * t;
      v[k] = (m(k, i) + m(i, k)) * t;
      x_ = v[0];
      y_ = v[1];
      z_ = v[2];
    }
  }
  T w() const { return w_; }
  T x() const { return x_; }
  T y() const { return y_; }
  T z() const { return z_; }
  Quaternion conjugate() const { return Quaternion(w_, -x_, -y_, -z_); }
  friend Quaternion operator*(const Quaternion& a, const Quaternion& b) {  // Hamilton product
    return Quaternion(a.w_ * b.w_ - a.x_ * b.x_ - a.y_ * b.y_ - a.z_ * b.z_,
                      a.w_ * b.x_ + a.x_ * b.w_ + a.y_ * b.z_ - a.z_ * b.y_,
                      a.w_ * b.y_ + a.y_ * b.w_ + a.z_ * b.x_ - a.x_ * b.z_,
                      a.w_ * b.z_ + a.z_ * b.w_ + a.x_ * b.y_ - a.y_ * b.x_);
  }

 private:
  T w_ = 1, x_ = 0, y_ = 0, z_ = 0;
};
using Quaterniond = Quaternion<double>;

// Umeyama (1991) similarity from src (3xN) to dst (3xN): 4x4 [cR | t; 0 1].
template <typename M>
Matrix<typename M::Scalar, 4, 4> umeyama(const M& src, const M& dst, bool with_scaling = true) {
  using T = typename M::Scalar;
  const Index n = src.cols();
  const T one_over_n = T(1) / static_cast<T>(n);
  Matrix<T, 3, 1> src_mean, dst_mean;
  for (Index i = 0; i < 3; ++i) {
    T a = src(i, 0), b = dst(i, 0);
    for (Index j = 1; j < n; ++j) {
      a = a + src(i, j);
      b = b + dst(i, j);
    }
    src_mean(i) = a * one_over_n;
    dst_mean(i) = b * one_over_n;
  }
  Matrix<T, 3, 3> sigma = Matrix<T, 3, 3>::Zero();
  T src_var = 0;
  for (Index j = 0; j < n; ++j) {
    Matrix<T, 3, 1> s, d;
    for (Index i = 0; i < 3; ++i) {
      s(i) = src(i, j) - src_mean(i);
      d(i) = dst(i, j) - dst_mean(i);
    }
    for (Index r = 0; r < 3; ++r)
      for (Index c = 0; c < 3; ++c) sigma(r, c) += d(r) * s(c);
    src_var += s.squaredNorm();
  }
  sigma = sigma * one_over_n;
  src_var = src_var * one_over_n;
  Matrix<T, 3, 3> u, v;
  Matrix<T, 3, 1> sv;
  detail::jacobi_svd_square<3>(sigma, &u, &sv, &v);
  Matrix<T, 3, 1> s = Matrix<T, 3, 1>::Constant(T(1));
  if (u.determinant() * v.determinant() < 0) s(2) = T(-1);
  Matrix<T, 3, 3> rot = u * s.asDiagonal() * v.transpose();
  Matrix<T, 4, 4> rt = Matrix<T, 4, 4>::Identity();
  T c = with_scaling ? T(1) / src_var * sv.dot(s) : T(1);
  Matrix<T, 3, 1> t = dst_mean - c * (rot * src_mean);
  for (Index r = 0; r < 3; ++r) {
    for (Index k = 0; k < 3; ++k) rt(r, k) = c * rot(r, k);
    rt(r, 3) = t(r);
  }
  return rt;
}

}  // namespace Eigen
