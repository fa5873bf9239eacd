"""Test-only CPU oracle (see gsopt_oracle.h). Never imported by the product."""
