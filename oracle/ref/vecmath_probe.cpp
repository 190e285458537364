// Probe of the tilesplat vecmath API (test infrastructure).  Compiled twice by
// oracle/ref/Makefile: against the reference header (/root/reference, when
// present) and against include/tilesplat/vecmath.hpp; tests compare the two
// outputs bit for bit.
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "tilesplat/vecmath.hpp"

using namespace tilesplat;

template <class T>
static void out(const char* tag, T v) {
    double d = double(v);
    uint64_t b;
    std::memcpy(&b, &d, 8);
    std::printf("%s %016llx\n", tag, (unsigned long long)b);
}

template <class T>
static void probe(const char* ty) {
    std::printf("# %s\n", ty);
    Vec2<T> a2{T(1.5), T(-2.25)}, b2{T(0.3), T(7)};
    out("v2.add", (a2 + b2).x), out("v2.sub", (a2 - b2).y), out("v2.mul", (a2 * T(1.7)).x);
    a2 += b2;
    out("v2.iadd", a2.y), out("v2.norm", a2.norm());
    Vec3<T> a{T(0.1), T(-3), T(2.5)}, b{T(4), T(0.7), T(-1.1)};
    out("v3.dot", a.dot(b)), out("v3.norm", a.norm()), out("v3.nz", a.normalized().z), out("v3.idx", a[2]);
    Vec3<T> c = a;
    c += b;
    c *= T(0.9);
    out("v3.c", c.x + c.y + c.z);
    Vec4<T> v4{T(1), T(2), T(-3), T(0.5)};
    v4[3] = T(4.25);
    out("v4.dot", v4.dot(v4)), out("v4.norm", v4.norm()), out("v4.idx", v4[3]);
    Quat<T> q{T(0.9), T(0.1), T(-0.3), T(0.2)};
    q[2] = T(-0.35);
    out("q.norm", q.norm()), out("q.sum", (q + q * T(0.5))[1]);
    Mat3<T> M = Mat3<T>::identity();
    M.m[0][1] = T(0.3), M.m[1][2] = T(-1.7), M.m[2][0] = T(2.2);
    Mat3<T> N = M * M.transposed();
    out("m3.mul", N.m[1][2]), out("m3.vec", (M * a).y), out("m3.tmul", M.transposed_mul(a).z);
    Mat2<T> P = Mat2<T>::identity();
    P.m[0][1] = T(0.5);
    out("m2.mul", (P * P).m[0][1]), out("m2.vec", (P * a2).x);
    Mat4<T> Q = Mat4<T>::identity();
    Q.m[0][3] = T(1.25), Q.m[2][1] = T(-0.75);
    out("m4.mul", (Q * Q.transposed()).m[0][0]), out("m4.vec", (Q * v4).z), out("m4.up", Q.upper3x3().m[2][1]);
    SymMat2<T> S{T(4), T(1.5), T(1)};
    SymMat2<T> S2 = S + S;
    S2 += S;
    out("s2.det", S.det()), out("s2.tr", S.trace()), out("s2.eig", S.max_eigenvalue()), out("s2.quad", S.quad(b2));
    out("s2.full", S2.full().m[1][0]);
    SymMat3<T> U{T(1), T(0.1), T(0.2), T(2), T(0.3), T(3)};
    out("s3.full", U.full().m[2][1]), out("s3.from", SymMat3<T>::from_full(N).yz), out("s3.sub", (U - U + U).zz);
    out("clamp", clamp(T(3.5), T(0), T(1))), out("clamp2", clamp(T(-2), T(-1), T(1)));
}

int main() {
    probe<float>("float");
    probe<double>("double");
    return 0;
}
