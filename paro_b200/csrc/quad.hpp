// Quadrature rules on the reference tetrahedron (host side): the reference's
// own nodes and weights (quad_tables.inc, see quad.cpp).
#pragma once

#include <array>
#include <vector>

namespace paro_b200 {

struct Rule {
  int degree = 1;
  std::vector<std::array<double, 4>> points;  // barycentric
  std::vector<double> weights;                // sum to 1
};

// simplex_rule(3, degree) (quadrature.cpp:169-177), degree 2 or 5
const Rule& simplex_rule3(int degree);
// subdivided_rule(3, degree, levels) (quadrature.cpp:179-188), (5, 2)
const Rule& subdivided_rule3(int degree, int levels);

}  // namespace paro_b200
