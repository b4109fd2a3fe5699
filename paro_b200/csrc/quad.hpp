// Quadrature rules on the reference tetrahedron (host side), restating
// proj/src/quadrature.cpp so the device sees identical nodes and weights.
#pragma once

#include <array>
#include <vector>

namespace paro_b200 {

struct Rule {
  int degree = 1;
  std::vector<std::array<double, 4>> points;  // barycentric
  std::vector<double> weights;                // sum to 1
};

// simplex_rule(3, degree) (quadrature.cpp:169-177 -> make_rule :80-108)
const Rule& simplex_rule3(int degree);
// subdivided_rule(3, degree, levels) (quadrature.cpp:179-188 -> make_subdivided :143-165)
const Rule& subdivided_rule3(int degree, int levels);

}  // namespace paro_b200
